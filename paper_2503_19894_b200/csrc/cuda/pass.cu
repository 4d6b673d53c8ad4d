// Launchers of the tile-pass kernel (kernels_pass.cuh) for both precisions.
//   complex128: tiles of 2^11 amplitudes, runs of 2^5  (32 KiB + 4 KiB pad per stage)
//   complex64 : tiles of 2^12 amplitudes, runs of 2^6  (32 KiB + 4 KiB pad per stage)
// Two CTAs of 256 threads per SM, two stages each: while one CTA's barriers
// hold its warps, the other's compute or copy.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "kernels_pass.cuh"

namespace tsg {
namespace {

void pass_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

template <typename Real, int M, int L>
int launch_pass_impl(const PassLaunch& pl, cudaStream_t s, int num_sms) {
  using S = PassShape<Real, M, L>;
  constexpr int kStages = 2;
  if (pl.tile_log2 != M || pl.run_log2 != L) throw std::runtime_error("pass geometry does not match the kernel");
  if (pl.n < M) throw std::runtime_error("state smaller than one pass tile");
  if (pl.blob_bytes % 16 != 0 || pl.blob_bytes > kPassMaxBlob) throw std::runtime_error("pass blob size");
  if (pl.n_ops <= 0) return 0;
  PassParams p{};
  p.re = pl.re;
  p.im = pl.im;
  p.blob = static_cast<const unsigned char*>(pl.blob);
  p.blob_bytes = pl.blob_bytes;
  p.n_ops = pl.n_ops;
  const int nh = M - L;
  int hp[16];
  for (int h = 0; h < nh; ++h) hp[h] = pl.high[h] - L;
  const int tile_bits = pl.n - M;
  p.n_tiles = uint64_t{1} << tile_bits;
  p.n_tmask = insertion_masks(hp, nh, tile_bits, p.tmask);
  if (p.n_tmask > kMaxMasks) throw std::runtime_error("pass tile masks");
  const size_t smem = S::smem_bytes(pl.blob_bytes, kStages);
  if (pl.jit) {  // the JIT-compiled kernel of this op table: same geometry, two CTAs per SM
    pass_check(cudaFuncSetAttribute(pl.jit, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "k_pass_jit smem attribute");
    int per_sm = 1;
    pass_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.jit, kPassThreads, smem), "k_pass_jit occupancy");
    const uint64_t blocks = std::min<uint64_t>(p.n_tiles, uint64_t(num_sms) * std::max(per_sm, 1));
    void* args[] = {&p};
    pass_check(cudaLaunchKernel(pl.jit, dim3(static_cast<unsigned>(blocks)), dim3(kPassThreads), args, smem, s),
               "k_pass_jit launch");
    return 1;
  }
  auto kern = k_pass<Real, M, L, kStages>;
  static size_t configured = 0;
  if (configured < smem) {
    pass_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "k_pass smem attribute");
    configured = smem;
  }
  int per_sm = 1;
  pass_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPassThreads, smem), "k_pass occupancy");
  const uint64_t blocks = std::min<uint64_t>(p.n_tiles, uint64_t(num_sms) * std::max(per_sm, 1));
  kern<<<static_cast<unsigned>(blocks), kPassThreads, smem, s>>>(p);
  pass_check(cudaGetLastError(), "k_pass launch");
  return 1;
}

}  // namespace

int launch_pass_f64(const PassLaunch& p, cudaStream_t s, int num_sms) { return launch_pass_impl<double, 11, 5>(p, s, num_sms); }
int launch_pass_f32(const PassLaunch& p, cudaStream_t s, int num_sms) { return launch_pass_impl<float, 12, 6>(p, s, num_sms); }

}  // namespace tsg
