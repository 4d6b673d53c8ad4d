// Probe: what cuTensorMapEncodeTiled accepts for the DMMA tile loads, and
// what the TMA unit does with it on B200.
//   A1  box dim 0 larger than the tensor's dim 0: padded chunks, OOB zeros
//   A2  a tile dimension (stride 2^L) aliasing the target dimensions
//   A3  tensor store of the A1 box: the padding must not be written
//   A4  a shared-memory destination 64 bytes past a 128-byte boundary (B200:
//       "misaligned address" -- tile destinations must be 128-byte aligned;
//       16 bytes past faults the same way)
// nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe scripts/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k_load(const __grid_constant__ CUtensorMap tm, int c0, int c1, int c2, int c3, int c4, int n, double* out,
                       int store, double* dst, int soff = 0) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  double* buf = reinterpret_cast<double*>(sm) + soff;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (store) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = -1.0 - i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile(
          "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(&tm),
          "r"(sa(buf)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) buf[i] = 12345.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(sa(buf)),
        "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(sa(&bar))
        : "memory");
    asm volatile(
        "{\n.reg .pred d;\nW: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n@!d bra W;\n}" ::"r"(sa(&bar))
        : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
}

static int make(CUtensorMap* tm, double* base, const uint64_t* dims, const uint64_t* strides_el, const uint32_t* box) {
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) gd[i] = dims[i], bx[i] = box[i];
  for (int i = 0; i < 4; ++i) gs[i] = strides_el[i] * 8;
  CUresult r = enc()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return static_cast<int>(r);
}

int main() {
  const int N = 1 << 16;
  std::vector<double> h(N);
  for (int i = 0; i < N; ++i) h[i] = i;
  double *d, *out;
  cudaMalloc(&d, N * 8);
  cudaMalloc(&out, 65536 * 8);
  cudaMemcpy(d, h.data(), N * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  int fails = 0;
  auto run = [&](const char* name, const uint64_t* dims, const uint64_t* st, const uint32_t* box, const int* c, int soff = 0) {
    CUtensorMap tm;
    int r = make(&tm, d, dims, st, box);
    printf("%s encode=%d\n", name, r);
    if (r) return;
    int n = box[0] * box[1] * box[2] * box[3] * box[4];
    k_load<<<1, 128, n * 8 + 1024>>>(tm, c[0], c[1], c[2], c[3], c[4], n, out, 0, nullptr, soff);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("  run error %s\n", cudaGetErrorString(e)); fails++; return; }
    std::vector<double> o(n);
    cudaMemcpy(o.data(), out, n * 8, cudaMemcpyDeviceToHost);
    int bad = 0, shown = 0;
    for (int i = 0; i < n; ++i) {
      int b[5], rem = i;
      for (int k = 0; k < 5; ++k) b[k] = rem % box[k], rem /= box[k];
      bool oob = false;
      int64_t a = 0;
      for (int k = 0; k < 5; ++k) {
        if (c[k] + b[k] >= static_cast<int64_t>(dims[k])) oob = true;
        a += (c[k] + b[k]) * (k ? st[k - 1] : 1);
      }
      double want = oob ? 0.0 : static_cast<double>(a);
      if (o[i] != want) { bad++; if (shown++ < 4) printf("  [%d] got %g want %g\n", i, o[i], want); }
    }
    printf("  %s: %d / %d mismatches\n", name, bad, n);
    fails += bad != 0;
  };
  {  // A1: 2048 chunks of 32, box 36 x 8 from chunk 5
    uint64_t dims[5] = {32, 2048, 1, 1, 1}, st[4] = {32, 65536, 65536, 65536};
    uint32_t box[5] = {36, 8, 1, 1, 1};
    int c[5] = {0, 5, 0, 0, 0};
    run("A1 oob-pad", dims, st, box, c);
  }
  {  // A2: runs of 64 (L = 6), tile dim stride 64 (size 1024), targets 11..15 (stride 2048, size 32)
    uint64_t dims[5] = {64, 1024, 32, 1, 1}, st[4] = {64, 2048, 65536, 65536};
    uint32_t box[5] = {68, 1, 32, 1, 1};
    int c[5] = {0, 31, 0, 0, 0};
    run("A2 alias", dims, st, box, c);
    int c2[5] = {0, 0b0000010000000000 >> 6 | 7, 0, 0, 0};
    run("A2b alias", dims, st, box, c2);
  }
  {  // A2c: strides not monotonic (target dim before the tile dim)
    uint64_t dims[5] = {64, 32, 1024, 1, 1}, st[4] = {2048, 64, 65536, 65536};
    uint32_t box[5] = {68, 32, 1, 1, 1};
    int c[5] = {0, 0, 31, 0, 0};
    run("A2c order", dims, st, box, c);
  }
  {  // A3: store the A1 box: padding must not be written
    uint64_t dims[5] = {32, 2048, 1, 1, 1}, st[4] = {32, 65536, 65536, 65536};
    uint32_t box[5] = {36, 8, 1, 1, 1};
    CUtensorMap tm;
    int r = make(&tm, d, dims, st, box);
    printf("A3 encode=%d\n", r);
    k_load<<<1, 128, 36 * 8 * 8>>>(tm, 0, 5, 0, 0, 0, 36 * 8, out, 1, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) printf("  run error %s\n", cudaGetErrorString(e));
    std::vector<double> o(N);
    cudaMemcpy(o.data(), d, N * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < N; ++i) {
      double want = i;
      int ch = i / 32, w = i % 32;
      if (ch >= 5 && ch < 13) want = -1.0 - ((ch - 5) * 36 + w);
      if (o[i] != want) { if (bad < 4) printf("  [%d] got %g want %g\n", i, o[i], want); bad++; }
    }
    printf("  A3 store: %d mismatches\n", bad);
    fails += bad != 0;
  }
  {  // A4 last: a misaligned destination is a sticky launch error
    uint64_t dims[5] = {32, 2048, 1, 1, 1}, st[4] = {32, 65536, 65536, 65536};
    uint32_t box[5] = {36, 8, 1, 1, 1};
    int c[5] = {0, 5, 0, 0, 0};
    run("A4 smem+64B (expected: misaligned address)", dims, st, box, c, 8);
  }
  printf("fails=%d\n", fails);
  return 0;
}
