// sm_100a gate-application kernels (the hot path).
//
// All kernels work in the s = 0 group space of the paper's GPU ABI
// (PAPER.md:371-380): group t in [0, 2^(n-k)), base = startIdx(t) computed
// with the SPEC mask table, then OR the active control
// values; the group's amplitudes sit at base + off[j], j < 2^ks.
//
//  k_direct  one thread per V groups; the 2^ks amplitudes of a group live in
//            registers, the snapped sub-matrix is a __grid_constant__ kernel
//            parameter (constant bank operands -- the GPU analogue of the
//            paper's -use-imm-value / -use-const-mem-space knobs).  SPARSE
//            skips Zero scalars with warp-uniform predicates.  HBM bound for
//            every ks where 2^ks complex FMAs per amplitude stay below the
//            FP64/FP32 ridge.
//  k_diag    diagonal sub-gates (CP, CZ, RZ, T, fused ZZ phases): a pure
//            stream over the active slice (controls fixed), 16-byte vector
//            loads, one read and one write per touched amplitude.
//  k_tile    ks = 5, 6: a CTA stages G groups x 2^ks amplitudes in shared
//            memory and computes the 2^ks x 2^ks by 2^ks x G product with a
//            register-blocked FMA micro-kernel (RT rows x GT groups / thread).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "gate_launch.hpp"

namespace tsg {

template <typename Real, int V>
struct VecOf;
template <>
struct VecOf<double, 1> {
  using T = double;
};
template <>
struct VecOf<double, 2> {
  using T = double2;
};
template <>
struct VecOf<float, 1> {
  using T = float;
};
template <>
struct VecOf<float, 2> {
  using T = float2;
};
template <>
struct VecOf<float, 4> {
  using T = float4;
};

template <typename Real, int V>
__device__ __forceinline__ void load_v(const Real* p, Real (&x)[V]) {
  using T = typename VecOf<Real, V>::T;
  const T v = *reinterpret_cast<const T*>(p);
  if constexpr (V == 1) {
    x[0] = v;
  } else if constexpr (V == 2) {
    x[0] = v.x;
    x[1] = v.y;
  } else {
    x[0] = v.x;
    x[1] = v.y;
    x[2] = v.z;
    x[3] = v.w;
  }
}

template <typename Real, int V>
__device__ __forceinline__ void store_v(Real* p, const Real (&x)[V]) {
  using T = typename VecOf<Real, V>::T;
  T v;
  if constexpr (V == 1) {
    v = x[0];
  } else if constexpr (V == 2) {
    v.x = x[0];
    v.y = x[1];
  } else {
    v.x = x[0];
    v.y = x[1];
    v.z = x[2];
    v.w = x[3];
  }
  *reinterpret_cast<T*>(p) = v;
}

// startIdx(t) = sum_i (t & masks[i]) << i
__device__ __forceinline__ uint64_t group_base(uint64_t t, const uint64_t* masks, int n_masks) {
  uint64_t b = 0;
#pragma unroll
  for (int i = 0; i < kMaxMasks; ++i)
    if (i < n_masks) b += (t & masks[i]) << i;
  return b;
}

// ------------------------------------------------------------------ direct
template <typename Real, int KS>
struct DirectParams {
  Real* re;
  Real* im;
  uint64_t g_begin;
  uint64_t n_work;  // number of V-group work items
  uint64_t fixed_or;
  uint64_t masks[kMaxMasks];
  int n_masks;
  uint32_t nz[((2 << (2 * KS)) + 31) / 32];  // scalar nonzero bits: 2e (re), 2e+1 (im)
  uint64_t off[1 << KS];
  Real mre[1 << (2 * KS)];
  Real mim[1 << (2 * KS)];
};

// Register budget: the 2^ks x V complex inputs of a work item stay in
// registers (at most 32 32-bit registers of inputs: V shrinks as ks grows);
// the 2^ks row addresses and the interleaved row accumulators need about as
// much again, so the occupancy floor drops from 4 to 1 CTA/SM with ks.
template <typename Real, int KS>
struct DirectShape {
  static constexpr int kRegsPerAmp = 2 * sizeof(Real) / 4;
  static constexpr int kAmpBudget = 32 / kRegsPerAmp;  // amplitudes per thread
  static constexpr int kVByBudget = kAmpBudget / (1 << KS);
  static constexpr int kVCap = sizeof(Real) == 8 ? (kVByBudget >= 2 ? 2 : 1)
                                                 : (kVByBudget >= 4 ? 4 : (kVByBudget >= 2 ? 2 : 1));
};
template <typename Real, int KS, int V>
struct DirectOcc {
  static constexpr int kMinBlocks = KS <= 2 ? 4 : (KS == 3 ? 2 : 1);
};

template <typename Real, int KS, int V, bool SPARSE>
__global__ void __launch_bounds__(256, (DirectOcc<Real, KS, V>::kMinBlocks)) k_direct(const __grid_constant__ DirectParams<Real, KS> p) {
  constexpr int D = 1 << KS;
  // One work item per thread and no grid-stride loop: a loop would let ptxas
  // hoist the 2*4^ks matrix scalars out of the constant bank into registers.
  const uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w < p.n_work) {
    const uint64_t base = group_base(p.g_begin + w * V, p.masks, p.n_masks) | p.fixed_or;
    Real xr[D][V], xi[D][V];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      load_v<Real, V>(p.re + base + p.off[j], xr[j]);
      load_v<Real, V>(p.im + base + p.off[j], xi[j]);
    }
#pragma unroll
    for (int r = 0; r < D; ++r) {
      Real yr[V], yi[V];
#pragma unroll
      for (int v = 0; v < V; ++v) yr[v] = yi[v] = Real(0);
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const int e = r * D + c;
        const Real ar = p.mre[e], ai = p.mim[e];
        if (!SPARSE || ((p.nz[(2 * e) >> 5] >> ((2 * e) & 31)) & 1u)) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            yr[v] = fma(ar, xr[c][v], yr[v]);
            yi[v] = fma(ar, xi[c][v], yi[v]);
          }
        }
        if (!SPARSE || ((p.nz[(2 * e + 1) >> 5] >> ((2 * e + 1) & 31)) & 1u)) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            yr[v] = fma(-ai, xi[c][v], yr[v]);
            yi[v] = fma(ai, xr[c][v], yi[v]);
          }
        }
      }
      store_v<Real, V>(p.re + base + p.off[r], yr);
      store_v<Real, V>(p.im + base + p.off[r], yi);
    }
  }
}

// -------------------------------------------------------------- diagonal
template <typename Real, int KD>
struct DiagParams {
  Real* re;
  Real* im;
  uint64_t n_work;  // (active elements) / V
  uint64_t fixed_or;
  int n_ctrl;
  int ctrl[12];  // ascending
  int tq[KD > 0 ? KD : 1];
  Real dre[1 << KD];
  Real dim[1 << KD];
};

__device__ __forceinline__ uint64_t insert_zero_bits(uint64_t x, const int* pos, int count) {
#pragma unroll
  for (int i = 0; i < 12; ++i)
    if (i < count) {
      const uint64_t low = x & ((uint64_t{1} << pos[i]) - 1);
      x = ((x ^ low) << 1) | low;
    }
  return x;
}

template <typename Real, int KD, int V>
__global__ void __launch_bounds__(256) k_diag(const __grid_constant__ DiagParams<Real, KD> p) {
  __shared__ Real sdr[1 << KD], sdi[1 << KD];
  for (int i = threadIdx.x; i < (1 << KD); i += blockDim.x) {
    sdr[i] = p.dre[i];
    sdi[i] = p.dim[i];
  }
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < p.n_work; w += stride) {
    const uint64_t idx = insert_zero_bits(w * V, p.ctrl, p.n_ctrl) | p.fixed_or;
    Real xr[V], xi[V];
    load_v<Real, V>(p.re + idx, xr);
    load_v<Real, V>(p.im + idx, xi);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      Real dr, di;
      if constexpr (KD == 0) {
        dr = p.dre[0];
        di = p.dim[0];
      } else {
        unsigned j = 0;
#pragma unroll
        for (int b = 0; b < KD; ++b) j |= static_cast<unsigned>(((idx + v) >> p.tq[b]) & 1u) << b;
        dr = sdr[j];
        di = sdi[j];
      }
      const Real r0 = xr[v], i0 = xi[v];
      xr[v] = fma(dr, r0, -di * i0);
      xi[v] = fma(dr, i0, di * r0);
    }
    store_v<Real, V>(p.re + idx, xr);
    store_v<Real, V>(p.im + idx, xi);
  }
}

// Diagonal sub-gates wider than k_diag's parameter table (7..12 qubits: a
// fused QAOA / IQP phase layer under the paper's k_max = 7 preset).  The
// 2^ks-entry table (fp64 re | im) is read through the read-only cache.  Full
// range: one thread per active amplitude.  Sub-range [g_begin, g_end) of the
// s = 0 group space: one thread per (group, entry).
template <typename Real>
struct DiagWideParams {
  Real* re;
  Real* im;
  const double* table;  // [2^ks re][2^ks im]
  uint64_t fixed_or;
  int n_ctrl, ks;
  int ctrl[12];  // ascending
  int tq[12];    // sub-target qubits, ascending
  bool full_range;
  uint64_t n_work;   // full range: active amplitudes; sub-range: groups x 2^ks
  uint64_t g_begin;  // sub-range: first group
  uint64_t masks[kMaxMasks];
  int n_masks;
};

template <typename Real>
__global__ void __launch_bounds__(256) k_diag_wide(const __grid_constant__ DiagWideParams<Real> p) {
  const uint64_t D = uint64_t{1} << p.ks;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < p.n_work; w += stride) {
    uint64_t idx;
    unsigned j = 0;
    if (p.full_range) {
      idx = insert_zero_bits(w, p.ctrl, p.n_ctrl) | p.fixed_or;
      for (int b = 0; b < p.ks; ++b) j |= static_cast<unsigned>((idx >> p.tq[b]) & 1u) << b;
    } else {
      j = static_cast<unsigned>(w & (D - 1));
      idx = group_base(p.g_begin + (w >> p.ks), p.masks, p.n_masks) | p.fixed_or;
      for (int b = 0; b < p.ks; ++b) idx |= static_cast<uint64_t>((j >> b) & 1u) << p.tq[b];
    }
    const Real dr = static_cast<Real>(__ldg(p.table + j)), di = static_cast<Real>(__ldg(p.table + D + j));
    const Real r0 = p.re[idx], i0 = p.im[idx];
    p.re[idx] = fma(dr, r0, -di * i0);
    p.im[idx] = fma(dr, i0, di * r0);
  }
}

// ------------------------------------------------------- diagonal batches
// One streaming pass applies a run of diagonal gates (DiagBatchLaunch).
template <typename Real>
struct Cplx2;
template <>
struct Cplx2<double> {
  using T = double2;
};
template <>
struct Cplx2<float> {
  using T = float2;
};

// Index arithmetic in 32 bits when the state has at most 2^32 amplitudes.
// A gate whose controls and targets avoid the V low bits has the same factor
// for all V amplitudes of a thread: it is resolved once per thread.
template <typename Real, int V, typename Idx>
__global__ void __launch_bounds__(256) k_diag_batch(const __grid_constant__ DiagBatchLaunch b, uint64_t n_work) {
  using C2 = typename Cplx2<Real>::T;
  __shared__ C2 tab[kMaxBatchEntries];
  for (int i = threadIdx.x; i < b.n_entries; i += blockDim.x)
    tab[i] = C2{static_cast<Real>(b.tables[2 * i]), static_cast<Real>(b.tables[2 * i + 1])};
  __syncthreads();
  Real* re = static_cast<Real*>(b.re);
  Real* im = static_cast<Real*>(b.im);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < n_work; w += stride) {
    const Idx idx0 = static_cast<Idx>(w * V);
    Real xr[V], xi[V];
    load_v<Real, V>(re + idx0, xr);
    load_v<Real, V>(im + idx0, xi);
    for (int g = 0; g < b.n_gates; ++g) {
      const Idx cm = static_cast<Idx>(b.cmask[g]), cv = static_cast<Idx>(b.cval[g]);
      const int ks = b.ks[g], off = b.toff[g];
      Idx tmask = 0;
      for (int t = 0; t < ks; ++t) tmask |= Idx{1} << b.tq[g][t];
      auto index_of = [&](Idx idx) {
        unsigned j = 0;
        for (int t = 0; t < ks; ++t) j |= static_cast<unsigned>(idx >> (b.tq[g][t] - t)) & (1u << t);
        return j;
      };
      auto apply = [&](int v, const C2 d) {
        const Real r0 = xr[v], i0 = xi[v];
        xr[v] = fma(d.x, r0, -d.y * i0);  // exactly k_diag's update
        xi[v] = fma(d.x, i0, d.y * r0);
      };
      if (((cm | tmask) & Idx{V - 1}) == 0) {  // same factor for the whole vector
        if ((idx0 & cm) != cv) continue;
        const C2 d = tab[off + index_of(idx0)];
#pragma unroll
        for (int v = 0; v < V; ++v) apply(v, d);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const Idx idx = idx0 + v;
          if ((idx & cm) == cv) apply(v, tab[off + index_of(idx)]);
        }
      }
    }
    store_v<Real, V>(re + idx0, xr);
    store_v<Real, V>(im + idx0, xi);
  }
}

// ------------------------------------------------------------------- tile
template <typename Real>
struct TileParams {
  Real* re;
  Real* im;
  const double* mat;  // [D*D re][D*D im][D*D re+im], row-major, FP64 for both precisions
  uint64_t g_begin, n_groups, n_tiles;
  uint64_t fixed_or;
  uint64_t masks[kMaxMasks];
  int n_masks;
  uint64_t off[1 << kMaxSub];
};

template <typename Real, int KS, int G, int RT, int GT>
struct TileShape {
  static constexpr int D = 1 << KS;
  static constexpr int kThreads = (D / RT) * (G / GT);
  static_assert(kThreads == 256, "tile shape must use 256 threads");
  static constexpr size_t kSmem = sizeof(Real) * (2 * D * G + 2 * D * D) + sizeof(uint64_t) * G;
};

template <typename Real, int KS, int G, int RT, int GT>
__global__ void __launch_bounds__(256) k_tile(const __grid_constant__ TileParams<Real> p) {
  using S = TileShape<Real, KS, G, RT, GT>;
  constexpr int D = S::D;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Real* Xr = reinterpret_cast<Real*>(smem_raw);  // [D][G]
  Real* Xi = Xr + D * G;
  Real* Mt = Xi + D * G;  // [D cols][D rows][2] : Mt[(c*D + r)*2 + {0,1}]
  uint64_t* bases = reinterpret_cast<uint64_t*>(Mt + 2 * D * D);

  for (int i = threadIdx.x; i < D * D; i += blockDim.x) {
    const int r = i / D, c = i % D;
    Mt[(c * D + r) * 2] = static_cast<Real>(p.mat[i]);
    Mt[(c * D + r) * 2 + 1] = static_cast<Real>(p.mat[D * D + i]);
  }
  const int gb = threadIdx.x % (G / GT);
  const int rb = threadIdx.x / (G / GT);

  for (uint64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const uint64_t t0 = p.g_begin + tile * G;
    const uint64_t g_lim = p.g_begin + p.n_groups;
    __syncthreads();  // previous tile's stores done with bases / X
    for (int g = threadIdx.x; g < G; g += blockDim.x)
      bases[g] = (t0 + g < g_lim) ? (group_base(t0 + g, p.masks, p.n_masks) | p.fixed_or) : ~uint64_t{0};
    __syncthreads();
    for (int i = threadIdx.x; i < D * G; i += blockDim.x) {
      const int j = i / G, g = i % G;
      const uint64_t b = bases[g];
      if (b != ~uint64_t{0}) {
        Xr[i] = p.re[b + p.off[j]];
        Xi[i] = p.im[b + p.off[j]];
      }
    }
    __syncthreads();
    Real ar[RT][GT], ai[RT][GT];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int g = 0; g < GT; ++g) ar[r][g] = ai[r][g] = Real(0);
#pragma unroll 4
    for (int c = 0; c < D; ++c) {
      Real xr[GT], xi[GT], mr[RT], mi[RT];
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        xr[g] = Xr[c * G + gb * GT + g];
        xi[g] = Xi[c * G + gb * GT + g];
      }
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        mr[r] = Mt[(c * D + rb * RT + r) * 2];
        mi[r] = Mt[(c * D + rb * RT + r) * 2 + 1];
      }
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int g = 0; g < GT; ++g) {
          ar[r][g] = fma(mr[r], xr[g], ar[r][g]);
          ar[r][g] = fma(-mi[r], xi[g], ar[r][g]);
          ai[r][g] = fma(mr[r], xi[g], ai[r][g]);
          ai[r][g] = fma(mi[r], xr[g], ai[r][g]);
        }
    }
    __syncthreads();  // every input consumed before the in-place write-back
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        Xr[(rb * RT + r) * G + gb * GT + g] = ar[r][g];
        Xi[(rb * RT + r) * G + gb * GT + g] = ai[r][g];
      }
    __syncthreads();
    for (int i = threadIdx.x; i < D * G; i += blockDim.x) {
      const int j = i / G, g = i % G;
      const uint64_t b = bases[g];
      if (b != ~uint64_t{0}) {
        p.re[b + p.off[j]] = Xr[i];
        p.im[b + p.off[j]] = Xi[i];
      }
    }
  }
}

}  // namespace tsg
