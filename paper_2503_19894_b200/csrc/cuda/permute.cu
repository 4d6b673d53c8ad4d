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
#include <type_traits>

#include "gate_launch.hpp"

namespace tsg {
namespace {

constexpr int kPermThreads = 256;
constexpr int kPermMaxTileLog2 = 10;
constexpr int kPermMaxTile = 1 << kPermMaxTileLog2;
constexpr int kPermPadded = kPermMaxTile + kPermMaxTile / 32;

__device__ __forceinline__ uint32_t perm_pad(uint32_t s) { return s + (s >> 5); }

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
  // pre-gate (PermuteLaunch::pre_*): its qubits as local tile bits
  int pre_k;  // <= 4
  int pre_lbit[4];       // local tile bit of sub-target bit b
  int pre_lbit_rank[4];  // the gate bit at the k-th gate position in ascending local order
  const double* pre_mat;  // [re | im] D x D row-major
};

// The pre-gate on the loaded tiles in shared memory.  Work items are (group,
// row) pairs spread over the CTA: phase 1 computes each item's output from
// the group's inputs (the row's nonzero entries only, staged in shared memory
// as a sparse row list), a barrier, phase 2 writes them in place.
constexpr int kPermPreItems = 2 * kPermMaxTile / kPermThreads;  // items per thread (two tiles)

constexpr int kPermPreMaxNnz = 128;  // nonzero entries of an absorbed gate (static shared memory budget)
struct PermPreRows {  // the pre-gate's rows, sparse (staged once per CTA)
  int start[17];      // row r: entries [start[r], start[r + 1])
  uint8_t col[kPermPreMaxNnz];
  double mr[kPermPreMaxNnz], mi[kPermPreMaxNnz];
};

template <typename Real>
__device__ __forceinline__ void perm_pre_gate(const PermParams& p, const PermPreRows& rows, Real (*tr)[kPermPadded],
                                              Real (*ti)[kPermPadded], int n_tiles) {
  const int K = p.pre_k, D = 1 << K, m = p.m;
  uint32_t gm = 0;  // local bits of the gate
  for (int b = 0; b < K; ++b) gm |= 1u << p.pre_lbit[b];
  auto local = [&](uint32_t g, uint32_t j) {  // deposit g over the non-gate bits, j over the gate bits
    uint32_t t = 0;
    for (int b = 0, kg = 0, kj = 0; b < m; ++b)
      if ((gm >> b) & 1u) t |= ((j >> p.pre_lbit_rank[kj++]) & 1u) << b;
      else t |= ((g >> kg++) & 1u) << b;
    return t;
  };
  const uint32_t items = static_cast<uint32_t>(n_tiles) << m;  // (tile, group, row): 2^m per tile
  Real yr[kPermPreItems], yi[kPermPreItems];
#pragma unroll
  for (int q = 0; q < kPermPreItems; ++q) {
    const uint32_t it = threadIdx.x + q * kPermThreads;
    yr[q] = yi[q] = Real(0);
    if (it >= items) continue;
    const int tile = static_cast<int>(it >> m);
    const uint32_t rest = it & ((1u << m) - 1), r = rest & (D - 1), g = rest >> K;
    for (int e = rows.start[r]; e < rows.start[r + 1]; ++e) {
      const uint32_t a = perm_pad(local(g, rows.col[e]));
      const Real mr = static_cast<Real>(rows.mr[e]), mi = static_cast<Real>(rows.mi[e]);
      const Real xr = tr[tile][a], xi = ti[tile][a];
      yr[q] = fma(mr, xr, yr[q]);
      yi[q] = fma(mr, xi, yi[q]);
      yr[q] = fma(-mi, xi, yr[q]);
      yi[q] = fma(mi, xr, yi[q]);
    }
  }
  __syncthreads();  // every item has read its group
#pragma unroll
  for (int q = 0; q < kPermPreItems; ++q) {
    const uint32_t it = threadIdx.x + q * kPermThreads;
    if (it >= items) continue;
    const int tile = static_cast<int>(it >> m);
    const uint32_t rest = it & ((1u << m) - 1), r = rest & (D - 1), g = rest >> K;
    const uint32_t a = perm_pad(local(g, r));
    tr[tile][a] = yr[q];
    ti[tile][a] = yi[q];
  }
}

template <typename Real, bool PRE>
__global__ void __launch_bounds__(kPermThreads, PRE ? 3 : 1) k_permute(const __grid_constant__ PermParams p) {
  // the pre-gate's sparse rows (a byte without a pre-gate: the plain kernel keeps its occupancy)
  __shared__ std::conditional_t<PRE, PermPreRows, char> pre_rows_storage;
  PermPreRows* pre_rows = reinterpret_cast<PermPreRows*>(&pre_rows_storage);
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
  if constexpr (PRE) {  // the pre-gate's nonzero entries, row by row
    if (threadIdx.x == 0) {
      const int D = 1 << p.pre_k;
      int e = 0;
      for (int r = 0; r < D; ++r) {
        pre_rows[0].start[r] = e;
        for (int c = 0; c < D; ++c) {
          const double mr = p.pre_mat[r * D + c], mi = p.pre_mat[D * D + r * D + c];
          if ((mr == 0.0 && mi == 0.0) || e >= kPermPreMaxNnz) continue;  // (the host bounds the count)
          pre_rows[0].col[e] = static_cast<uint8_t>(c);
          pre_rows[0].mr[e] = mr;
          pre_rows[0].mi[e] = mi;
          ++e;
        }
      }
      pre_rows[0].start[D] = e;
    }
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
    if constexpr (PRE) {  // the absorbed gate, on each loaded tile before the permutation
      // (its own instantiation: the plain permutation keeps its registers and occupancy)
      perm_pre_gate<Real>(p, pre_rows[0], tr, ti, self ? 1 : 2);
      __syncthreads();
    }
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

// tile bits: the run bits, their images, then the preferred qubits (a
// pre-gate's) with their images, then further p-closed positions
int perm_tile_bits(const int* p, int n, bool* in_t, uint64_t prefer = 0) {
  const int m_target = std::min(kPermMaxTileLog2, n);
  int m = 0;
  for (int q = 0; q < std::min(5, n); ++q) {
    for (int r : {q, p[q]})
      if (!in_t[r]) {
        in_t[r] = true;
        ++m;
      }
  }
  for (int q = 0; q < n && m < m_target; ++q) {
    if (!((prefer >> q) & 1u) || in_t[q]) continue;
    const int need = p[q] == q ? 1 : 2;
    if (m + need > m_target) continue;
    in_t[q] = in_t[p[q]] = true;
    m += need;
  }
  for (int q = 0; q < n && m < m_target; ++q) {
    if (in_t[q]) continue;
    const int need = p[q] == q ? 1 : 2;
    if (m + need > m_target) continue;
    in_t[q] = in_t[p[q]] = true;
    m += need;
  }
  return m;
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
  bool in_t[64] = {};
  uint64_t prefer = 0;
  for (int b = 0; b < pl.pre_k; ++b) prefer |= uint64_t{1} << pl.pre_q[b];
  const int m = perm_tile_bits(pl.p, n, in_t, prefer);
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
  if (pl.pre_k > 4) throw std::runtime_error("k_permute: pre-gate wider than 4 qubits");
  p.pre_k = pl.pre_k;
  p.pre_mat = pl.pre_mat;
  for (int b = 0; b < pl.pre_k; ++b) {
    if (pl.pre_q[b] < 0 || pl.pre_q[b] >= n || !in_t[pl.pre_q[b]]) throw std::runtime_error("k_permute: pre-gate off the tile");
    p.pre_lbit[b] = lpos[pl.pre_q[b]];
  }
  for (int k = 0; k < pl.pre_k; ++k) {  // gate bits by ascending local position
    int rank = 0;
    for (int b = 0; b < pl.pre_k; ++b) rank += p.pre_lbit[b] < p.pre_lbit[k];
    p.pre_lbit_rank[rank] = k;
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
  auto kern = pl.pre_k > 0 ? k_permute<Real, true> : k_permute<Real, false>;
  int per_sm = 1;
  perm_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPermThreads, 0), "k_permute occupancy");
  const uint64_t blocks = std::min<uint64_t>(p.n_units, uint64_t(num_sms) * std::max(per_sm, 1) * 4);
  kern<<<static_cast<unsigned>(blocks), kPermThreads, 0, s>>>(p);
  perm_check(cudaGetLastError(), "k_permute launch");
  return 1;
}

}  // namespace

uint64_t permute_tile_mask(const int* p, int n, uint64_t prefer) {
  bool in_t[64] = {};
  perm_tile_bits(p, n, in_t, prefer);
  uint64_t mask = 0;
  for (int q = 0; q < n; ++q) mask |= static_cast<uint64_t>(in_t[q]) << q;
  return mask;
}

int launch_permute_f64(const PermuteLaunch& p, cudaStream_t s, int num_sms) { return launch_permute_impl<double>(p, s, num_sms); }
int launch_permute_f32(const PermuteLaunch& p, cudaStream_t s, int num_sms) { return launch_permute_impl<float>(p, s, num_sms); }

}  // namespace tsg
