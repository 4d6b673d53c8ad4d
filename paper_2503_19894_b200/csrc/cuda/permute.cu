// k_permute: an involutive permutation of the qubits (bit positions) of the
// state, in place, in one HBM sweep.
//
// new[y] = old[P(y)], P moving bit q of the index to position p[q] with
// p[p[q]] = q (a product of disjoint qubit swaps, e.g. QFT's bit-reversal
// layer; a general qubit permutation is two of these, runtime.cu).  Tiles:
// the tile bits T are the low run bits A = [0, 5) plus their images p(A)
// (padded with further p-closed positions to 2^10 amplitudes); every other
// bit is fixed within a tile and P maps tile c to tile P(c).  A CTA takes the
// pair {c, P(c)} (c <= P(c)): loads both tiles (32-amplitude contiguous runs,
// coalesced), gathers tile P(c)'s amplitudes into tile c's order through
// shared memory and vice versa, and stores both (again whole runs).  Tiles
// mapped to themselves are permuted within the tile.  Shared-memory rows are
// padded by one element per 32 so the gather along permuted bits spreads
// over the banks.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "gate_launch.hpp"

namespace tsg {
namespace {

constexpr int kPermThreads = 256;
constexpr int kPermMaxTileLog2 = 10;
constexpr int kPermMaxTile = 1 << kPermMaxTileLog2;
constexpr int kPermPadded = kPermMaxTile + kPermMaxTile / 32;

struct PermParams {
  void* re;
  void* im;
  int m;                          // tile bits
  uint64_t n_units;               // 2^(n - m) tiles
  uint64_t omask[kMaxMasks + 8];  // insertion masks: unit index -> its index bits (zeros at T)
  int n_omask;
  int n_mo;                       // moved positions outside the tile
  int mo_from[64], mo_to[64];
  uint64_t mo_mask;
  uint64_t tdep[kPermMaxTileLog2];  // local tile bit i -> index bit
  int tsrc[kPermMaxTileLog2];       // local tile bit i -> local position of P's image
};

__device__ __forceinline__ uint32_t perm_pad(uint32_t s) { return s + (s >> 5); }

template <typename Real>
__global__ void __launch_bounds__(kPermThreads) k_permute(const __grid_constant__ PermParams p) {
  __shared__ uint64_t dep[kPermMaxTile];   // local index t -> index bits
  __shared__ uint16_t src[kPermMaxTile];   // local index t -> padded smem slot of its source
  __shared__ Real tr[2][kPermPadded], ti[2][kPermPadded];
  const int tile = 1 << p.m;
  for (int t = threadIdx.x; t < tile; t += kPermThreads) {
    uint64_t d = 0;
    uint32_t s = 0;
    for (int i = 0; i < p.m; ++i)
      if ((t >> i) & 1) {
        d |= p.tdep[i];
        s |= 1u << p.tsrc[i];
      }
    dep[t] = d;
    src[t] = static_cast<uint16_t>(perm_pad(s));
  }
  __syncthreads();
  Real* re = static_cast<Real*>(p.re);
  Real* im = static_cast<Real*>(p.im);
  for (uint64_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
    uint64_t c = 0;
    for (int i = 0; i < p.n_omask; ++i) c += (u & p.omask[i]) << i;
    uint64_t pc = c & ~p.mo_mask;
    for (int i = 0; i < p.n_mo; ++i) pc |= ((c >> p.mo_from[i]) & 1u) << p.mo_to[i];
    if (pc < c) continue;  // the pair is the partner's
    const bool self = pc == c;
    for (int t = threadIdx.x; t < tile; t += kPermThreads) {
      const uint64_t d = dep[t];
      const uint32_t w = perm_pad(t);
      tr[0][w] = re[c | d];
      ti[0][w] = im[c | d];
      if (!self) {
        tr[1][w] = re[pc | d];
        ti[1][w] = im[pc | d];
      }
    }
    __syncthreads();
    const int other = self ? 0 : 1;
    for (int t = threadIdx.x; t < tile; t += kPermThreads) {
      const uint64_t d = dep[t];
      const uint32_t s = src[t];
      re[c | d] = tr[other][s];
      im[c | d] = ti[other][s];
      if (!self) {
        re[pc | d] = tr[0][s];
        im[pc | d] = ti[0][s];
      }
    }
    __syncthreads();
  }
}

void perm_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

template <typename Real>
int launch_permute_impl(const PermuteLaunch& pl, cudaStream_t s, int num_sms) {
  const int n = pl.n;
  bool any = false;
  for (int q = 0; q < n; ++q) {
    if (pl.p[q] < 0 || pl.p[q] >= n || pl.p[pl.p[q]] != q) throw std::runtime_error("k_permute: not an involution");
    any |= pl.p[q] != q;
  }
  if (!any) return 0;
  // tile bits: the run bits, their images, then further p-closed positions
  const int m_target = std::min(kPermMaxTileLog2, n);
  bool in_t[64] = {};
  int m = 0;
  for (int q = 0; q < std::min(5, n); ++q) {
    for (int r : {q, pl.p[q]})
      if (!in_t[r]) {
        in_t[r] = true;
        ++m;
      }
  }
  for (int q = 0; q < n && m < m_target; ++q) {
    if (in_t[q]) continue;
    const int need = pl.p[q] == q ? 1 : 2;
    if (m + need > m_target) continue;
    in_t[q] = in_t[pl.p[q]] = true;
    m += need;
  }
  if (m > kPermMaxTileLog2) throw std::runtime_error("k_permute: tile too large");
  PermParams p{};
  p.re = pl.re;
  p.im = pl.im;
  p.m = m;
  int tpos[64], lpos[64], nt = 0, opos[64], no = 0;
  for (int q = 0; q < n; ++q) {
    if (in_t[q]) {
      lpos[q] = nt;
      tpos[nt++] = q;
    } else {
      opos[no++] = q;
    }
  }
  for (int i = 0; i < m; ++i) {
    p.tdep[i] = uint64_t{1} << tpos[i];
    p.tsrc[i] = lpos[pl.p[tpos[i]]];
  }
  p.n_units = uint64_t{1} << (n - m);
  p.n_omask = insertion_masks(tpos, m, n - m, p.omask);
  for (int i = 0; i < no; ++i)
    if (pl.p[opos[i]] != opos[i]) {
      p.mo_from[p.n_mo] = opos[i];
      p.mo_to[p.n_mo] = pl.p[opos[i]];
      p.mo_mask |= uint64_t{1} << opos[i];
      ++p.n_mo;
    }
  int per_sm = 1;
  perm_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_permute<Real>, kPermThreads, 0), "k_permute occupancy");
  const uint64_t blocks = std::min<uint64_t>(p.n_units, uint64_t(num_sms) * std::max(per_sm, 1) * 4);
  k_permute<Real><<<static_cast<unsigned>(blocks), kPermThreads, 0, s>>>(p);
  perm_check(cudaGetLastError(), "k_permute launch");
  return 1;
}

}  // namespace

int launch_permute_f64(const PermuteLaunch& p, cudaStream_t s, int num_sms) { return launch_permute_impl<double>(p, s, num_sms); }
int launch_permute_f32(const PermuteLaunch& p, cudaStream_t s, int num_sms) { return launch_permute_impl<float>(p, s, num_sms); }

}  // namespace tsg
