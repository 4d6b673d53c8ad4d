// k_stream: persistent, TMA-pipelined gate kernel for sub-gates of 3..5 qubits.
//
// Tile geometry (host side: stream_geometry() in runtime.cu).  Index bits
// [0, L) form the "lower region" (SPEC.md:412-417 with s = L: the GPU version
// of the paper's shuffled loading); L is chosen so that a tile
// holds G = 2^(L - #targets below L) whole groups.  A tile is the 2^{k_Hs}
// runs of 2^L contiguous amplitudes selected by the high sub-target bits
// (high controls fixed at their active value), so every global access is a
// contiguous >= 256-byte bulk copy regardless of where the targets sit:
//
//   tile t:   base(t) = deposit(t over non-target bits >= L) | ctrl bits
//   run r:    base(t) + roff[r]                 r < 2^{k_Hs}
//   smem:     stage[s] = run_0 | run_1 | ...    (re and im arrays)
//   group g:  lbase(g) = deposit(g over non-target bits < L) | low ctrl bits
//   element j of group g  = smem[lbase(g) + soff[j]]
//
// Pipeline: one elected thread issues cp.async.bulk global->shared copies for
// S stages (mbarrier complete_tx), the CTA computes stage i while stages
// i+1..i+S-1 land, writes results in place, fences the async proxy and bulk-
// stores the runs back (cp.async.bulk shared->global, bulk_group).
//
// Compute: warp (wr, wg) owns rows [8 wr, 8 wr + 8) of the 2^ks x 2^ks sub-
// matrix for 32 groups (lanes); the row block is a compile-time constant per
// switch arm, so matrix scalars are constant-bank operands.  Complex MACs use
// the 3-multiplication form: S1 += c a, S2 += d b, S3 += (c+d)(a+b);
// re = S1 - S2, im = S3 - S1 - S2 (3 FMAs instead of 4; zero scalars skip
// their FMA in the SPARSE variant, which is exactly zero-skipping).
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>

#include <cuda_runtime.h>
#endif

#include "gate_launch.hpp"

namespace tsg {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
// TMA tensor-map copies (cp.async.bulk.tensor, SASS UTMALDG / UTMASTG): the
// descriptor is an opaque 128-byte CUtensorMap built on the host
// (cuTensorMapEncodeTiled) and passed inside a __grid_constant__ parameter
// block; every copy here is rank 5 with only coordinate 2 nonzero.
struct alignas(64) TmaDesc {
  unsigned long long w[16];
};
__device__ __forceinline__ void tma_g2s(void* dst, const TmaDesc* d, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %2, %3, %2, "
      "%2}], [%4];" ::"r"(smem_addr(dst)),
      "l"(d), "r"(0), "r"(c2), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_s2g(const TmaDesc* d, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %2, %3, %2, %2}], [%1];" ::"l"(d),
               "r"(smem_addr(src)), "r"(0), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------ shape
template <int KS>
struct StreamShape {
  static constexpr int D = 1 << KS;
  static constexpr int RW = D < 8 ? D : 8;          // rows per warp
  static constexpr int WR = D / RW;                 // warps across rows
  static constexpr int WG = WR >= 4 ? 1 : 4 / WR;   // warps across groups
  static constexpr int W = WR * WG;
  static constexpr int kThreads = 32 * W;
  static constexpr int P = 2;                       // passes of 32*WG groups per tile
  static constexpr int G = P * 32 * WG;             // groups per tile
  static constexpr int LOG2G = KS == 3 ? 8 : (KS == 4 ? 7 : 6);
  static_assert((1 << LOG2G) == G, "group count must be a power of two");
};

template <typename Real, int KS>
struct StreamParams {
  Real* re;
  Real* im;
  uint64_t n_tiles;
  uint64_t ctrl_or;  // active control values (absolute bit positions)
  uint64_t tmask[kMaxMasks];  // tile id -> bits >= L (pre-shift) with high targets inserted
  int n_tmask;
  int L;
  int n_runs;
  uint32_t gmask[kMaxMasks];  // group id -> bits < L with low targets inserted
  int n_gmask;
  uint64_t roff[1 << KS];
  uint32_t soff[1 << KS];
  uint32_t nz[(3 << (2 * KS)) / 32 + 1];  // SPARSE: bits 3e (re), 3e+1 (im), 3e+2 (re+im)
  Real mr[1 << (2 * KS)];
  Real mi[1 << (2 * KS)];
  Real ms[1 << (2 * KS)];  // mr + mi for the 3-multiplication form
};

template <typename Real, int KS>
__device__ __forceinline__ uint64_t stream_tile_base(const StreamParams<Real, KS>& p, uint64_t tile) {
  uint64_t b = 0;
#pragma unroll
  for (int i = 0; i < kMaxMasks; ++i)
    if (i < p.n_tmask) b += (tile & p.tmask[i]) << i;
  // only the controls above the lower region select runs; low controls are
  // folded into the group base inside the tile
  return (b << p.L) | (p.ctrl_or & ~((uint64_t{1} << p.L) - 1));
}

template <typename Real, int KS>
__device__ __forceinline__ uint32_t stream_group_base(const StreamParams<Real, KS>& p, uint32_t g) {
  uint32_t b = 0;
#pragma unroll
  for (int i = 0; i < kMaxMasks; ++i)
    if (i < p.n_gmask) b += (g & p.gmask[i]) << i;
  return b | static_cast<uint32_t>(p.ctrl_or & ((uint64_t{1} << p.L) - 1));
}

template <typename Real, int KS, int WRI, bool SPARSE>
__device__ __forceinline__ void stream_rows(const StreamParams<Real, KS>& p, const Real* xr, const Real* xi,
                                            uint32_t lb, Real (&orr)[StreamShape<KS>::RW],
                                            Real (&oii)[StreamShape<KS>::RW]) {
  using S = StreamShape<KS>;
  Real s1[S::RW], s2[S::RW], s3[S::RW];
#pragma unroll
  for (int r = 0; r < S::RW; ++r) s1[r] = s2[r] = s3[r] = Real(0);
#pragma unroll
  for (int c = 0; c < S::D; ++c) {
    const Real a = xr[lb + p.soff[c]];
    const Real b = xi[lb + p.soff[c]];
    const Real ab = a + b;
#pragma unroll
    for (int r = 0; r < S::RW; ++r) {
      const int e = (WRI * S::RW + r) * S::D + c;
      if (!SPARSE || ((p.nz[(3 * e) >> 5] >> ((3 * e) & 31)) & 1u)) s1[r] = fma(p.mr[e], a, s1[r]);
      if (!SPARSE || ((p.nz[(3 * e + 1) >> 5] >> ((3 * e + 1) & 31)) & 1u)) s2[r] = fma(p.mi[e], b, s2[r]);
      if (!SPARSE || ((p.nz[(3 * e + 2) >> 5] >> ((3 * e + 2) & 31)) & 1u)) s3[r] = fma(p.ms[e], ab, s3[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < S::RW; ++r) {
    orr[r] = s1[r] - s2[r];
    oii[r] = s3[r] - s1[r] - s2[r];
  }
}

template <typename Real, int KS, bool SPARSE>
__device__ __forceinline__ void stream_rows_dispatch(int wr, const StreamParams<Real, KS>& p, const Real* xr,
                                                     const Real* xi, uint32_t lb, Real (&orr)[StreamShape<KS>::RW],
                                                     Real (&oii)[StreamShape<KS>::RW]) {
  using S = StreamShape<KS>;
  if constexpr (S::WR == 1) {
    stream_rows<Real, KS, 0, SPARSE>(p, xr, xi, lb, orr, oii);
  } else if constexpr (S::WR == 2) {
    if (wr == 0) stream_rows<Real, KS, 0, SPARSE>(p, xr, xi, lb, orr, oii);
    else stream_rows<Real, KS, 1, SPARSE>(p, xr, xi, lb, orr, oii);
  } else {
    static_assert(S::WR == 4, "row split");
    switch (wr) {
      case 0: stream_rows<Real, KS, 0, SPARSE>(p, xr, xi, lb, orr, oii); break;
      case 1: stream_rows<Real, KS, 1, SPARSE>(p, xr, xi, lb, orr, oii); break;
      case 2: stream_rows<Real, KS, 2, SPARSE>(p, xr, xi, lb, orr, oii); break;
      default: stream_rows<Real, KS, 3, SPARSE>(p, xr, xi, lb, orr, oii); break;
    }
  }
}

template <typename Real, int KS, int STAGES, bool SPARSE>
__global__ void __launch_bounds__(StreamShape<KS>::kThreads) k_stream(const __grid_constant__ StreamParams<Real, KS> p) {
  using S = StreamShape<KS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t run_len = 1u << p.L;
  const uint32_t tile_elems = run_len * static_cast<uint32_t>(p.n_runs);
  Real* buf = reinterpret_cast<Real*>(smem_raw);  // [STAGES][2][tile_elems]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(Real) * 2 * STAGES * tile_elems);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = warp / S::WG, wg = warp % S::WG;
  const uint32_t stage_bytes = 2 * tile_elems * sizeof(Real);
  const uint32_t run_bytes = run_len * sizeof(Real);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto issue_load = [&](uint64_t tile, int s) {
    const uint64_t base = stream_tile_base(p, tile);
    Real* dr = buf + (2 * s) * tile_elems;
    Real* di = dr + tile_elems;
    mbar_expect_tx(&bars[s], stage_bytes);
    for (int r = 0; r < p.n_runs; ++r) {
      bulk_g2s(dr + r * run_len, p.re + base + p.roff[r], run_bytes, &bars[s]);
      bulk_g2s(di + r * run_len, p.im + base + p.roff[r], run_bytes, &bars[s]);
    }
  };

  const uint64_t first = blockIdx.x, step = gridDim.x;
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s)
      if (first + s * step < p.n_tiles) issue_load(first + s * step, s);

  uint32_t it = 0;
  for (uint64_t tile = first; tile < p.n_tiles; tile += step, ++it) {
    const int s = static_cast<int>(it % STAGES);
    if (tid == 0 && it > 0) {
      // stage of iteration it-1 is free once its bulk store has read smem
      bulk_wait_read_all();
      const uint64_t next = tile + (STAGES - 1) * step;
      if (next < p.n_tiles) issue_load(next, static_cast<int>((it + STAGES - 1) % STAGES));
    }
    mbar_wait(&bars[s], (it / STAGES) & 1u);
    Real* xr = buf + (2 * s) * tile_elems;
    Real* xi = xr + tile_elems;

    Real orr[S::P][S::RW], oii[S::P][S::RW];
    uint32_t lbs[S::P];
#pragma unroll
    for (int q = 0; q < S::P; ++q) {
      const uint32_t g = static_cast<uint32_t>((q * S::WG + wg) * 32 + lane);
      lbs[q] = stream_group_base(p, g);
      stream_rows_dispatch<Real, KS, SPARSE>(wr, p, xr, xi, lbs[q], orr[q], oii[q]);
    }
    __syncthreads();  // every warp has read the stage: results may overwrite it
#pragma unroll
    for (int q = 0; q < S::P; ++q)
#pragma unroll
      for (int r = 0; r < S::RW; ++r) {
        const uint32_t a = lbs[q] + p.soff[wr * S::RW + r];
        xr[a] = orr[q][r];
        xi[a] = oii[q][r];
      }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const uint64_t base = stream_tile_base(p, tile);
      for (int r = 0; r < p.n_runs; ++r) {
        bulk_s2g(p.re + base + p.roff[r], xr + r * run_len, run_bytes);
        bulk_s2g(p.im + base + p.roff[r], xi + r * run_len, run_bytes);
      }
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
}

}  // namespace tsg
