// k_stream_dmma: complex128 sub-gates of 3..5 qubits on the FP64 tensor pipe.
//
// Same tile pipeline as k_stream (kernels_stream.cuh: runs of 2^L contiguous
// amplitudes, cp.async.bulk global<->shared, mbarrier stages, persistent CTAs)
// but the product Y = M X per tile (M: D x D sub-matrix, X: D x G groups) is
// computed with mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), which on B200 runs at
// the full FP64 rate (measured 63.6 MAC/clk/SM, scripts/microbench.cu) while
// keeping M in registers for the whole persistent kernel -- constant-bank
// operands fall to 27-46 DFMA/clk/SM once the matrix exceeds ~2 KB.
//
// Fragments (PTX m8n8k4 .f64; lr = lane/4, lc = lane%4):
//   A (8x4 row) = M[8 rb + lr][4 ks + lc]        held in registers
//   B (4x8 col) = X[4 ks + lc][8 nb + lr]         one LDS.64 each (re, im)
//   C (8x8)     = Y[8 rb + lr][8 nb + 2 lc + i]   i = 0, 1
// Complex product with three real products (3M): T1 = Mr Xr, T2 = Mi Xi,
// T3 = (Mr + Mi)(Xr + Xi); Yr = T1 - T2, Yi = T3 - T1 - T2.  An 8x4 block of
// Mr / Mi / Ms that is all zero skips its DMMA (warp-uniform), which is the
// block form of SPEC's zero-skipping.
//
// Runs are laid out in shared memory with a stride of 2^L + 8 doubles so the
// four k-rows of a B fragment (different runs when the targets are high) fall
// in different bank halves: each LDS.64 costs the minimum two wavefronts.
#pragma once

#include <cstdint>

#include "kernels_stream.cuh"

namespace tsg {

constexpr int kRunPad = 8;  // doubles between runs in shared memory

template <int KS>
struct DmmaShape {
  static constexpr int D = 1 << KS;
  static constexpr int RB = D / 8;               // 8-row blocks
  static constexpr int WR = RB;                  // one warp per row block
  static constexpr int WG = RB >= 4 ? 1 : 4 / RB;
  static constexpr int W = WR * WG;
  static constexpr int kThreads = 32 * W;
  static constexpr int G = 64;                   // groups per tile
  static constexpr int LOG2G = 6;
  static constexpr int GW = G / WG;              // groups per warp
  static constexpr int NR = GW / 8;              // 8-group blocks per warp
  static constexpr int KST = D / 4;              // k-steps
};

template <int KS>
struct DmmaParams {
  double* re;
  double* im;
  const double* mat;  // [Mr | Mi | Ms], each D x D row-major (device)
  uint64_t n_tiles;
  uint64_t ctrl_hi;   // active control values at or above bit L
  uint32_t ctrl_lo;   // active control values below bit L
  uint64_t tmask[kMaxMasks];
  int n_tmask;
  int L;
  int n_runs;
  uint32_t run_stride;  // 2^L + kRunPad
  uint32_t gmask[kMaxMasks];
  int n_gmask;
  uint64_t roff[1 << KS];  // global offset of run r
  uint32_t soff[1 << KS];  // shared offset of element j (padded runs)
  uint32_t nzblk[3];       // bit (rb * KST + ks): block of Mr / Mi / Ms is nonzero
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int KS>
__device__ __forceinline__ uint32_t dmma_group_base(const DmmaParams<KS>& p, uint32_t g) {
  uint32_t b = 0;
#pragma unroll
  for (int i = 0; i < kMaxMasks; ++i)
    if (i < p.n_gmask) b += (g & p.gmask[i]) << i;
  return b | p.ctrl_lo;
}

template <int KS, int STAGES, bool SPARSE>
__global__ void __launch_bounds__(DmmaShape<KS>::kThreads) k_stream_dmma(const __grid_constant__ DmmaParams<KS> p) {
  using S = DmmaShape<KS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t run_len = 1u << p.L;
  const uint32_t stage_elems = p.run_stride * static_cast<uint32_t>(p.n_runs);
  double* buf = reinterpret_cast<double*>(smem_raw);  // [STAGES][2][stage_elems]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(double) * 2 * STAGES * stage_elems);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int rb = warp / S::WG, wg = warp % S::WG;
  const int lr = lane >> 2, lc = lane & 3;
  const uint32_t run_bytes = run_len * sizeof(double);

  // M fragments for this warp's row block, for the kernel's lifetime
  double amr[S::KST], ami[S::KST], ams[S::KST];
  constexpr int DD = S::D * S::D;
#pragma unroll
  for (int k = 0; k < S::KST; ++k) {
    const int e = (8 * rb + lr) * S::D + 4 * k + lc;
    amr[k] = p.mat[e];
    ami[k] = p.mat[DD + e];
    ams[k] = p.mat[2 * DD + e];
  }
  // per-thread shared offsets: B rows, C rows, group bases (tile independent)
  uint32_t offb[S::KST], lbb[S::NR], lbc[S::NR][2];
#pragma unroll
  for (int k = 0; k < S::KST; ++k) offb[k] = p.soff[4 * k + lc];
  const uint32_t offc = p.soff[8 * rb + lr];
#pragma unroll
  for (int nb = 0; nb < S::NR; ++nb) {
    const uint32_t g0 = wg * S::GW + nb * 8;
    lbb[nb] = dmma_group_base(p, g0 + lr);
    lbc[nb][0] = dmma_group_base(p, g0 + 2 * lc);
    lbc[nb][1] = dmma_group_base(p, g0 + 2 * lc + 1);
  }

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto tile_base = [&](uint64_t tile) {
    uint64_t b = 0;
#pragma unroll
    for (int i = 0; i < kMaxMasks; ++i)
      if (i < p.n_tmask) b += (tile & p.tmask[i]) << i;
    return (b << p.L) | p.ctrl_hi;
  };
  auto issue_load = [&](uint64_t tile, int s) {
    const uint64_t base = tile_base(tile);
    double* dr = buf + (2 * s) * stage_elems;
    double* di = dr + stage_elems;
    mbar_expect_tx(&bars[s], 2u * run_bytes * static_cast<uint32_t>(p.n_runs));
    for (int r = 0; r < p.n_runs; ++r) {
      bulk_g2s(dr + r * p.run_stride, p.re + base + p.roff[r], run_bytes, &bars[s]);
      bulk_g2s(di + r * p.run_stride, p.im + base + p.roff[r], run_bytes, &bars[s]);
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
      bulk_wait_read_all();  // the previous stage's bulk store has read smem
      const uint64_t next = tile + (STAGES - 1) * step;
      if (next < p.n_tiles) issue_load(next, static_cast<int>((it + STAGES - 1) % STAGES));
    }
    mbar_wait(&bars[s], (it / STAGES) & 1u);
    double* xr = buf + (2 * s) * stage_elems;
    double* xi = xr + stage_elems;

    double t1[S::NR][2], t2[S::NR][2], t3[S::NR][2];
#pragma unroll
    for (int nb = 0; nb < S::NR; ++nb) t1[nb][0] = t1[nb][1] = t2[nb][0] = t2[nb][1] = t3[nb][0] = t3[nb][1] = 0.0;
#pragma unroll
    for (int k = 0; k < S::KST; ++k) {
      const int bit = rb * S::KST + k;
      const bool use_r = !SPARSE || ((p.nzblk[0] >> bit) & 1u);
      const bool use_i = !SPARSE || ((p.nzblk[1] >> bit) & 1u);
      const bool use_s = !SPARSE || ((p.nzblk[2] >> bit) & 1u);
#pragma unroll
      for (int nb = 0; nb < S::NR; ++nb) {
        const double br = xr[lbb[nb] + offb[k]];
        const double bi = xi[lbb[nb] + offb[k]];
        if (use_r) dmma(t1[nb], amr[k], br);
        if (use_i) dmma(t2[nb], ami[k], bi);
        if (use_s) dmma(t3[nb], ams[k], br + bi);
      }
    }
    __syncthreads();  // every warp has read the stage: write results in place
#pragma unroll
    for (int nb = 0; nb < S::NR; ++nb)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint32_t a = lbc[nb][i] + offc;
        xr[a] = t1[nb][i] - t2[nb][i];
        xi[a] = t3[nb][i] - t1[nb][i] - t2[nb][i];
      }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const uint64_t base = tile_base(tile);
      for (int r = 0; r < p.n_runs; ++r) {
        bulk_s2g(p.re + base + p.roff[r], xr + r * p.run_stride, run_bytes);
        bulk_s2g(p.im + base + p.roff[r], xi + r * p.run_stride, run_bytes);
      }
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
}

}  // namespace tsg
