// k_stream_dmma: complex128 sub-gates of 3..6 qubits on the FP64 tensor pipe.
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
// Runs are laid out in shared memory with a stride of 2^L + 4 doubles: 64-bit
// shared loads are served per half-warp, and a stride of 8 banks puts the four
// k-rows of a B fragment (different runs when the targets are high) in four
// distinct bank quarters, so each LDS.64 costs the minimum two wavefronts.
//
// Warp roles: warp W (the last) is the producer -- its lanes issue the bulk
// loads of a stage (full[s] mbarrier, complete_tx) and, for ks <= 4, the bulk
// stores of its results once empty[s] says every consumer warp is done with
// it; warps 0..W-1 wait on full[s] and run the DMMA product.  For ks = 5 the
// consumers arrive on empty[s] as soon as they have read the stage and store
// their results straight from the accumulator fragments to global memory
// (the FP64-bound case: a stage is free for the next load sooner); for
// ks <= 4 they write the results into the stage (in place) for the bulk store.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#include <type_traits>
#endif

#include "kernels_stream.cuh"

namespace tsg {

// padding between runs in shared memory: 32 bytes = 8 banks, so the four
// k-rows of a B fragment land in distinct bank quarters (both precisions)
constexpr int kRunPadBytes = 32;

// A tile holds 2^AMPS_LOG2 amplitudes (2048 for complex128, 4096 for
// complex64 -- the per-tile pipeline latency is roughly fixed, so tiles are
// sized in amplitudes, measured); every consumer warp owns 8 n-blocks of 8
// groups for one 8-row block.
template <int KS, int AMPS_LOG2 = 11, int NRB = 8>
struct DmmaShape {
  static constexpr int D = 1 << KS;
  static constexpr int RB = D / 8;               // 8-row blocks
  static constexpr int WR = RB;                  // one warp per row block
  static constexpr int LOG2G = AMPS_LOG2 - KS;   // groups per tile
  static constexpr int G = 1 << LOG2G;
  static constexpr int NR = NRB;                 // 8-group blocks per warp
  static constexpr int GW = 8 * NR;              // groups per warp
  static constexpr int WG = G / GW;              // warps across groups
  static constexpr int W = WR * WG;
  static constexpr int kThreads = 32 * W;
  static constexpr int KST = D / 4;              // k-steps
  static_assert(WG >= 1, "tile too small");
};
// 8 n-blocks per warp where registers allow; 4 for the widest sub-gates so
// that 16 consumer warps fit per SM (DMMA issue needs the warps).
#ifndef TSG_D5_AMPS
#define TSG_D5_AMPS 11
#endif
#ifndef TSG_D5_NRB
#define TSG_D5_NRB 4
#endif
// complex128 6-qubit products: 2048-amplitude tiles (32 groups), 2 n-blocks
// per warp, so 16 consumer warps share the SM's one CTA (the M fragments take
// 96 KB of shared memory)
#ifndef TSG_D6_NRB
#define TSG_D6_NRB 2
#endif
template <typename Real, int KS>
using DShape = DmmaShape<KS, sizeof(Real) == 8 ? (KS == 5 ? TSG_D5_AMPS : 11) : 12,
                         (sizeof(Real) == 8 && KS == 5)   ? TSG_D5_NRB
                         : (sizeof(Real) == 8 && KS == 6) ? TSG_D6_NRB
                                                          : ((KS >= 5 || (sizeof(Real) == 4 && KS >= 4)) ? 4 : 8)>;

// Real = storage type of the state (double: complex128, float: complex64);
// the product always runs in FP64 on the DMMA pipe (complex64 amplitudes are
// widened on load and rounded once on store).
template <typename Real, int KS>
struct DmmaParams {
  Real* re;
  Real* im;
  const double* mat;  // [Mr | Mi | Ms], each D x D row-major (device)
  uint64_t n_tiles;
  uint64_t ctrl_hi;   // active control values at or above bit L
  uint32_t ctrl_lo;   // active control values below bit L
  uint64_t tmask[kMaxMasks];
  int n_tmask;
  int L;
  int n_runs;
  uint32_t run_stride;  // shared-memory elements per run (padded)
  // A run is stored as 2^(L - chunk_log2) chunks of 2^chunk_log2 amplitudes,
  // chunk_stride elements apart (chunk_log2 = L: one padded chunk per run).
  // Chunking spreads runs whose groups would all start on the same bank.
  int chunk_log2;
  uint32_t chunk_stride;
  uint32_t gmask[kMaxMasks];
  int n_gmask;
  uint64_t roff[1 << KS];  // global offset of run r
  uint32_t soff[1 << KS];  // shared offset of element j (padded runs and chunks)
  uint64_t goff[1 << KS];  // global offset of element j from the tile base
  uint32_t nzblk[3];       // bit (rb * KST + ks): block of Mr / Mi / Ms is nonzero
  uint32_t stage_elems;    // shared elements per array and stage (a multiple of 128 bytes)
  // TMA tensor-map tile copies (dmma_tma_plan; tma_issues = 0: one bulk copy
  // per chunk).  The maps view re / im as [chunk + pad | chunks per run |
  // tile (stride 2^L) | run bits | run bits]; copy i moves runs
  // [i << tma_shift, (i + 1) << tma_shift) at tile coordinate
  // (base + roff[i << tma_shift]) >> L, tma_issue_elems shared elements apart.
  int tma_issues;
  int tma_store;  // write-back through the maps too (else per-chunk bulk stores)
  int tma_shift;
  uint32_t tma_issue_elems;
  TmaDesc tmap[2];
};

// A pure function of its operands (no volatile): the compiler may schedule
// the fragment loads around it freely.
#ifndef TSG_DMMA_VOLATILE
#define TSG_DMMA_VOLATILE 0
#endif
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
#if TSG_DMMA_VOLATILE
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
#else
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
#endif
}

// in-run position of group g (low targets zero, low controls at their value)
template <typename Real, int KS>
__device__ __forceinline__ uint32_t dmma_group_pos(const DmmaParams<Real, KS>& p, uint32_t g) {
  uint32_t b = 0;
#pragma unroll
  for (int i = 0; i < kMaxMasks; ++i)
    if (i < p.n_gmask) b += (g & p.gmask[i]) << i;
  return b | p.ctrl_lo;
}

// shared-memory offset of an in-run position (chunk padding; additive over disjoint bits)
template <typename Real, int KS>
__device__ __forceinline__ uint32_t dmma_pad(const DmmaParams<Real, KS>& p, uint32_t w) {
  return (w >> p.chunk_log2) * p.chunk_stride + (w & ((1u << p.chunk_log2) - 1));
}

// M fragments live in registers for ks <= 4; for ks = 5, 6 they are staged in
// shared memory in fragment order ([3][KST][RB][32 lanes], conflict-free
// LDS.64): 24 KB for ks = 5 (the consumer warps fit 2 CTAs per SM), 96 KB for
// ks = 6 (one CTA per SM).  ks = 6 runs dense only: its 128 tiles per matrix
// do not fit nzblk's 32-bit masks.
template <int KS>
__host__ __device__ constexpr bool dmma_m_in_regs() {
  return KS <= 4;
}
// shared memory ahead of the stages: M fragments (FP64 DMMA, ks = 5) or the
// sub-matrix as {re, im} FP32 pairs (SIMT: complex64 3-qubit sub-gates with
// every target and control at bit 5 or above -- FP32 FMA at twice the FP64
// rate, lanes on contiguous groups; measured faster than the FP64-widened
// DMMA product there, slower for 4-5 qubits and low targets)
template <typename Real, int KS, bool SIMT = false>
__host__ __device__ constexpr size_t dmma_m_smem_bytes() {
  if (SIMT) return size_t{8} << (2 * KS);
  return dmma_m_in_regs<KS>() ? 0 : size_t{3} * ((1 << KS) / 4) * ((1 << KS) / 8) * 32 * sizeof(double);
}

// Tile bases in the persistent order first, first + step, ...: stepped in
// the masked domain (non-tile bits forced to 1 so the carry crosses them).
struct DmmaTileStream {
  uint64_t raw, mask, dstep, ctrl;
  __device__ uint64_t base() const { return raw | ctrl; }
  __device__ void advance() { raw = ((raw | ~mask) + dstep) & mask; }
};

// Which 8 x 4 tiles of Mr / Mi / Ms the product visits: all (dense), the
// launch's runtime masks (p.nzblk, per-tile predicates), or masks compiled
// into a JIT kernel (DmmaStaticNz: the skipped DMMAs and loads vanish from
// the code; per row block the consumer loop is instantiated once).
struct DmmaDenseNz {
  static constexpr bool kStatic = true, kDense = true;
  template <typename P>
  static __device__ __forceinline__ constexpr bool use(const P&, int, int) { return true; }
};
struct DmmaRuntimeNz {
  static constexpr bool kStatic = false, kDense = false;
  template <typename P>
  static __device__ __forceinline__ bool use(const P& p, int m, int bit) { return (p.nzblk[m] >> bit) & 1u; }
};
template <uint32_t M0, uint32_t M1, uint32_t M2>
struct DmmaStaticNz {
  static constexpr bool kStatic = true, kDense = false;
  template <typename P>
  static __device__ __forceinline__ constexpr bool use(const P&, int m, int bit) {
    return (((m == 0 ? M0 : (m == 1 ? M1 : M2)) >> bit) & 1u) != 0;
  }
};

// Consumer warps of k_stream_dmma: Y = M X on the DMMA pipe for row block RB
// (RBC >= 0: a compile-time row block, RBC < 0: rb at run time).
// TPOSE (direct-out only): the product is computed transposed, Y^T = X^T M^T
// -- the same fragment registers with the mma operands swapped -- so that a
// lane holds two ADJACENT elements of one group instead of one element of
// two groups: with qubit 0 as the first element bit (targets on qubit 0,
// where two groups are never adjacent) every store is a 2-element vector.
template <typename Real, int KS, int STAGES, typename NZ, bool MREG, bool kDirectOut, int RBC, bool TPOSE = false>
__device__ __forceinline__ void dmma_consumer(const DmmaParams<Real, KS>& p, Real* buf, uint64_t* full, uint64_t* empty,
                                              uint32_t stage_elems, const double* mfrag,
                                              const DmmaTileStream& stream0, int warp_rb, int wg, int lane) {
  using S = DShape<Real, KS>;
  const int rb = RBC >= 0 ? RBC : warp_rb;
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const int lr = lane >> 2, lc = lane & 3;
  double amr[MREG ? S::KST : 1], ami[MREG ? S::KST : 1], ams[MREG ? S::KST : 1];
  if constexpr (MREG) {
    constexpr int DD = S::D * S::D;
#pragma unroll
    for (int k = 0; k < S::KST; ++k) {
      const int e = (8 * rb + lr) * S::D + 4 * k + lc;
      amr[k] = p.mat[e];
      ami[k] = p.mat[DD + e];
      ams[k] = p.mat[2 * DD + e];
    }
  }
  const double* mf = mfrag + rb * 32 + lane;  // fragment (m, k) at mf[(m * KST + k) * RB * 32]
  uint32_t offb[S::KST], lbb[S::NR], lbc[S::NR][2];
#pragma unroll
  for (int k = 0; k < S::KST; ++k) offb[k] = p.soff[4 * k + lc];
  // output row 8 rb + lr: shared offset offc (ks <= 4 write-back) and global
  // offset goffc from the tile base (ks = 5 stores from registers); a
  // group's base is padded for shared memory (lbb, lbc) and raw for global
  // memory (gbc)
  const uint32_t offc = p.soff[8 * rb + lr];
  const uint64_t goffc = p.goff[8 * rb + lr];
  uint32_t gbc[S::NR][2];
#pragma unroll
  for (int nb = 0; nb < S::NR; ++nb) {
    const uint32_t g0 = wg * S::GW + nb * 8;
    lbb[nb] = dmma_pad(p, dmma_group_pos(p, g0 + lr));
    gbc[nb][0] = dmma_group_pos(p, g0 + 2 * lc);
    gbc[nb][1] = dmma_group_pos(p, g0 + 2 * lc + 1);
    lbc[nb][0] = dmma_pad(p, gbc[nb][0]);
    lbc[nb][1] = dmma_pad(p, gbc[nb][1]);
  }
  // no target on bit 0: groups 2c, 2c+1 are adjacent, even-aligned amplitudes
  const bool pair_store = gbc[0][1] == gbc[0][0] + 1 && (gbc[0][0] & 1u) == 0 && (goffc & 1u) == 0;
  // transposed: this lane's elements 8 rb + 2 lc (+1) of group 8 nb + lr
  static_assert(!TPOSE || kDirectOut, "transposed products store from registers");
  const uint64_t goffe = p.goff[8 * rb + 2 * lc];
  const bool pair_store_t = p.goff[8 * rb + 2 * lc + 1] == goffe + 1 && (goffe & 1u) == 0;
  uint32_t gbt[S::NR];
#pragma unroll
  for (int nb = 0; nb < S::NR; ++nb) gbt[nb] = dmma_group_pos(p, wg * S::GW + nb * 8 + lr);

  DmmaTileStream cstream = stream0;  // output addresses (ks = 5)
  uint32_t j = 0;
  for (uint64_t tile = first; tile < p.n_tiles; tile += step, ++j) {
    const int s = static_cast<int>(j % STAGES);
    mbar_wait(&full[s], (j / STAGES) & 1u);
    Real* xr = buf + (2 * s) * stage_elems;
    Real* xi = xr + stage_elems;

    double t1[S::NR][2], t2[S::NR][2], t3[S::NR][2];
#pragma unroll
    for (int nb = 0; nb < S::NR; ++nb) t1[nb][0] = t1[nb][1] = t2[nb][0] = t2[nb][1] = t3[nb][0] = t3[nb][1] = 0.0;
#pragma unroll
    for (int k = 0; k < S::KST; ++k) {
      const int bit = rb * S::KST + k;
      const bool use_r = NZ::use(p, 0, bit);
      const bool use_i = NZ::use(p, 1, bit);
      const bool use_s = NZ::use(p, 2, bit);
      if (!(use_r || use_i || use_s)) continue;  // zero k-step of this row block: no loads either
      // (compiled-in masks drop the loads of unused operands too; runtime
      // masks load every operand of an active k-step)
      constexpr bool kDrop = NZ::kStatic;
      double fr = 0.0, fi = 0.0, fs = 0.0;
      if constexpr (MREG) {
        fr = amr[k];
        fi = ami[k];
        fs = ams[k];
      } else {
        if (!kDrop || use_r) fr = mf[(0 * S::KST + k) * S::RB * 32];
        if (!kDrop || use_i) fi = mf[(1 * S::KST + k) * S::RB * 32];
        if (!kDrop || use_s) fs = mf[(2 * S::KST + k) * S::RB * 32];
      }
#pragma unroll
      for (int nb = 0; nb < S::NR; ++nb) {
        const double br = (!kDrop || use_r || use_s) ? static_cast<double>(xr[lbb[nb] + offb[k]]) : 0.0;
        const double bi = (!kDrop || use_i || use_s) ? static_cast<double>(xi[lbb[nb] + offb[k]]) : 0.0;
        if constexpr (TPOSE) {  // C^T = B^T A^T: the B fragment serves as A and vice versa
          if (use_r) dmma(t1[nb], br, fr);
          if (use_i) dmma(t2[nb], bi, fi);
          if (use_s) dmma(t3[nb], br + bi, fs);
        } else {
          if (use_r) dmma(t1[nb], fr, br);
          if (use_i) dmma(t2[nb], fi, bi);
          if (use_s) dmma(t3[nb], fs, br + bi);
        }
      }
    }
    if constexpr (!kDirectOut) {
      // all consumer warps have read the stage before anyone overwrites it
      asm volatile("bar.sync 1, %0;" ::"r"(S::kThreads) : "memory");
#pragma unroll
      for (int nb = 0; nb < S::NR; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const uint32_t a = lbc[nb][i] + offc;
          xr[a] = static_cast<Real>(t1[nb][i] - t2[nb][i]);
          xi[a] = static_cast<Real>(t3[nb][i] - t1[nb][i] - t2[nb][i]);
        }
      fence_async_smem();  // generic-proxy writes -> async-proxy bulk store
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[s])) : "memory");
      continue;
    }
    // this warp has read the stage: release it to the producer, then write
    // the results from registers (the stage is not written back)
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[s])) : "memory");
    if constexpr (TPOSE) {
      const uint64_t tbe = cstream.base() + goffe;
      cstream.advance();
      using V2 = std::conditional_t<sizeof(Real) == 8, double2, float2>;
#pragma unroll
      for (int nb = 0; nb < S::NR; ++nb) {
        const uint64_t a = tbe + gbt[nb];
        const Real r0 = static_cast<Real>(t1[nb][0] - t2[nb][0]), r1 = static_cast<Real>(t1[nb][1] - t2[nb][1]);
        const Real i0 = static_cast<Real>(t3[nb][0] - t1[nb][0] - t2[nb][0]);
        const Real i1 = static_cast<Real>(t3[nb][1] - t1[nb][1] - t2[nb][1]);
        if (pair_store_t) {
          *reinterpret_cast<V2*>(p.re + a) = V2{r0, r1};
          *reinterpret_cast<V2*>(p.im + a) = V2{i0, i1};
        } else {
          p.re[a] = r0;
          p.im[a] = i0;
          const uint64_t b = a - goffe + p.goff[8 * rb + 2 * lc + 1];
          p.re[b] = r1;
          p.im[b] = i1;
        }
      }
      continue;
    }
    const uint64_t tb = cstream.base() + goffc;
    cstream.advance();
    if (pair_store) {  // the lane's two groups are adjacent amplitudes: one 2-element store per array
#pragma unroll
      for (int nb = 0; nb < S::NR; ++nb) {
        const uint64_t a = tb + gbc[nb][0];
        using V2 = std::conditional_t<sizeof(Real) == 8, double2, float2>;
        *reinterpret_cast<V2*>(p.re + a) = V2{static_cast<Real>(t1[nb][0] - t2[nb][0]), static_cast<Real>(t1[nb][1] - t2[nb][1])};
        *reinterpret_cast<V2*>(p.im + a) = V2{static_cast<Real>(t3[nb][0] - t1[nb][0] - t2[nb][0]),
                                              static_cast<Real>(t3[nb][1] - t1[nb][1] - t2[nb][1])};
      }
    } else {
#pragma unroll
      for (int nb = 0; nb < S::NR; ++nb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const uint64_t a = tb + gbc[nb][i];
          p.re[a] = static_cast<Real>(t1[nb][i] - t2[nb][i]);
          p.im[a] = static_cast<Real>(t3[nb][i] - t1[nb][i] - t2[nb][i]);
        }
    }
  }
}

template <typename Real, int KS, int STAGES, bool SPARSE, bool SIMT, typename NZ, bool TPOSE = false>
__device__ __forceinline__ void k_stream_dmma_body(const DmmaParams<Real, KS>& p) {
  using S = DShape<Real, KS>;
  constexpr bool MREG = dmma_m_in_regs<KS>();
  // ks = 5 (FP64-bound): results leave from registers so a stage frees as soon
  // as it is read; ks <= 4 (HBM-bound): in-place smem write-back + bulk stores
  // (full 256-byte+ runs) measured faster
#ifndef TSG_DMMA_DIRECT_OUT_MIN_KS
#define TSG_DMMA_DIRECT_OUT_MIN_KS 5
#endif
  constexpr bool kSimt = SIMT;
#ifndef TSG_DMMA_DIRECT_OUT_MIN_KS_F32
#define TSG_DMMA_DIRECT_OUT_MIN_KS_F32 4
#endif
  // (complex64 4-qubit products are FP64-bound too: widened to the DMMA pipe)
  constexpr bool kDirectOut =
      KS >= (sizeof(Real) == 4 ? TSG_DMMA_DIRECT_OUT_MIN_KS_F32 : TSG_DMMA_DIRECT_OUT_MIN_KS) && !kSimt;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t stage_elems = p.stage_elems;
  double* mfrag = reinterpret_cast<double*>(smem_raw);  // [3][KST][RB][32] when !MREG
  Real* buf = reinterpret_cast<Real*>(smem_raw + dmma_m_smem_bytes<Real, KS, SIMT>());  // [STAGES][2][stage_elems]
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(buf) +
                                               sizeof(Real) * 2 * STAGES * stage_elems);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int chunk_shift = p.L - p.chunk_log2;  // chunks per run = 2^chunk_shift
  const int n_chunks = p.n_runs << chunk_shift;
  const uint32_t chunk_bytes = (1u << p.chunk_log2) * sizeof(Real);
  const uint64_t first = blockIdx.x, step = gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], S::W);
    }
    mbar_fence_init();
  }
  if constexpr (kSimt) {
    constexpr int DD = S::D * S::D;
    float2* smat = reinterpret_cast<float2*>(smem_raw);
    for (int i = tid; i < DD; i += blockDim.x) smat[i] = float2{static_cast<float>(p.mat[i]), static_cast<float>(p.mat[DD + i])};
  } else if constexpr (!MREG) {
    constexpr int DD = S::D * S::D;
    constexpr int NF = 3 * S::KST * S::RB * 32;
    for (int f = tid; f < NF; f += blockDim.x) {
      const int ln = f % 32, rbf = (f / 32) % S::RB, k = (f / (32 * S::RB)) % S::KST, m = f / (32 * S::RB * S::KST);
      mfrag[f] = p.mat[m * DD + (8 * rbf + (ln >> 2)) * S::D + 4 * k + (ln & 3)];
    }
  }
  __syncthreads();

  auto raw_base = [&](uint64_t tile) {
    uint64_t b = 0;
#pragma unroll
    for (int i = 0; i < kMaxMasks; ++i)
      if (i < p.n_tmask) b += (tile & p.tmask[i]) << i;
    return b << p.L;
  };
  const DmmaTileStream stream0{raw_base(first), raw_base(p.n_tiles - 1), raw_base(step), p.ctrl_hi};

  if (warp == S::W) {
    // ---------------- producer warp: TMA bulk loads and stores ------------
    // Copies are spread over the 32 lanes (lane l owns runs l, l+32, ...);
    // bulk groups are per thread, so every lane waits for its own stores.
    DmmaTileStream lstream = stream0, sstream = stream0;  // next tile to load / to store
    auto load = [&](uint64_t tile, int s) {
      const uint64_t base = lstream.base();
      lstream.advance();
      Real* dr = buf + (2 * s) * stage_elems;
      Real* di = dr + stage_elems;
      if (p.tma_issues > 0) {  // a few tensor copies per tile (padding included)
        if (lane == 0) {
          mbar_expect_tx(&full[s], 2u * sizeof(Real) * p.run_stride * static_cast<uint32_t>(p.n_runs));
          for (int i = 0; i < p.tma_issues; ++i) {
            const int c2 = static_cast<int>((base + p.roff[i << p.tma_shift]) >> p.L);
            tma_g2s(dr + i * p.tma_issue_elems, &p.tmap[0], c2, &full[s]);
            tma_g2s(di + i * p.tma_issue_elems, &p.tmap[1], c2, &full[s]);
          }
        }
        return;
      }
      if (lane == 0) mbar_expect_tx(&full[s], 2u * chunk_bytes * static_cast<uint32_t>(n_chunks));
      __syncwarp();
      for (int c = lane; c < n_chunks; c += 32) {
        const int r = c >> chunk_shift, q = c & ((1 << chunk_shift) - 1);
        const uint32_t so = r * p.run_stride + q * p.chunk_stride;
        const uint64_t go = base + p.roff[r] + (static_cast<uint64_t>(q) << p.chunk_log2);
        bulk_g2s(dr + so, p.re + go, chunk_bytes, &full[s]);
        bulk_g2s(di + so, p.im + go, chunk_bytes, &full[s]);
      }
    };
    for (int s = 0; s < STAGES; ++s)
      if (first + s * step < p.n_tiles) load(first + s * step, s);
    uint32_t j = 0;
    for (uint64_t tile = first; tile < p.n_tiles; tile += step, ++j) {
      const int s = static_cast<int>(j % STAGES);
      const uint64_t next = tile + STAGES * step;
      if constexpr (kDirectOut) {
        if (next >= p.n_tiles) break;
        mbar_wait(&empty[s], (j / STAGES) & 1u);  // the consumers have read tile j
        load(next, s);
      } else {
        mbar_wait(&empty[s], (j / STAGES) & 1u);  // the consumers wrote tile j's results
        const uint64_t base = sstream.base();
        sstream.advance();
        const Real* sr = buf + (2 * s) * stage_elems;
        const Real* si = sr + stage_elems;
        if (p.tma_store) {
          if (lane == 0)
            for (int i = 0; i < p.tma_issues; ++i) {
              const int c2 = static_cast<int>((base + p.roff[i << p.tma_shift]) >> p.L);
              tma_s2g(&p.tmap[0], c2, sr + i * p.tma_issue_elems);
              tma_s2g(&p.tmap[1], c2, si + i * p.tma_issue_elems);
            }
        } else {
          for (int c = lane; c < n_chunks; c += 32) {
            const int r = c >> chunk_shift, q = c & ((1 << chunk_shift) - 1);
            const uint32_t so = r * p.run_stride + q * p.chunk_stride;
            const uint64_t go = base + p.roff[r] + (static_cast<uint64_t>(q) << p.chunk_log2);
            bulk_s2g(p.re + go, sr + so, chunk_bytes);
            bulk_s2g(p.im + go, si + so, chunk_bytes);
          }
        }
        bulk_commit();
        if (next < p.n_tiles) {
          bulk_wait_read_all();  // this lane's stores have read the stage
          __syncwarp();
          load(next, s);
        }
      }
    }
    if constexpr (!kDirectOut) bulk_wait_all();
    return;
  }

  if constexpr (kSimt) {
    // ---------------- consumer warps, complex64: FP32 SIMT product ---------
    // Thread t owns GP groups (t, t + T, ...) when the tile has more groups
    // than threads, else group t % G and rows [RS (t / G), RS (t / G) + RS).
    // Lanes take consecutive groups: every element load of a warp is one
    // contiguous run of the stage; matrix entries are warp-uniform broadcasts.
    constexpr int T = S::kThreads, G = S::G, D = S::D;
    constexpr int GP = G >= T ? G / T : 1;
    constexpr int RS = G >= T ? D : D * G / T;
    const float2* smat = reinterpret_cast<const float2*>(smem_raw);
    const int r0 = G >= T ? 0 : (tid / G) * RS;
    uint32_t gb[GP];
#pragma unroll
    for (int q = 0; q < GP; ++q) gb[q] = dmma_pad(p, dmma_group_pos(p, (G >= T ? tid : tid % G) + q * T));
    uint32_t jt = 0;
    for (uint64_t tile = first; tile < p.n_tiles; tile += step, ++jt) {
      const int s = static_cast<int>(jt % STAGES);
      mbar_wait(&full[s], (jt / STAGES) & 1u);
      Real* xr = buf + (2 * s) * stage_elems;
      Real* xi = xr + stage_elems;
      float yr[GP][RS], yi[GP][RS];
#pragma unroll
      for (int q = 0; q < GP; ++q) {
        float vr[D], vi[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          vr[j] = xr[gb[q] + p.soff[j]];
          vi[j] = xi[gb[q] + p.soff[j]];
        }
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          float ar = 0.f, ai = 0.f;
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const float2 m = smat[(r0 + r) * D + c];
            ar = fmaf(m.x, vr[c], ar);
            ai = fmaf(m.x, vi[c], ai);
            ar = fmaf(-m.y, vi[c], ar);
            ai = fmaf(m.y, vr[c], ai);
          }
          yr[q][r] = ar;
          yi[q][r] = ai;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");  // every consumer has read the stage
#pragma unroll
      for (int q = 0; q < GP; ++q)
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          const uint32_t a = gb[q] + p.soff[r0 + r];
          xr[a] = yr[q][r];
          xi[a] = yi[q][r];
        }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[s])) : "memory");
    }
    return;
  }

  // ---------------- consumer warps: Y = M X on the DMMA pipe --------------
  const int rb = warp / S::WG, wg = warp % S::WG;
  if constexpr (NZ::kStatic && !NZ::kDense) {
    // compiled-in masks: one straight-line product per row block
    static_assert(S::RB <= 8, "row blocks");
#define TSG_DMMA_RB(R)                                                                                          \
  if constexpr (S::RB > R)                                                                                      \
    if (rb == R) return dmma_consumer<Real, KS, STAGES, NZ, MREG, kDirectOut, R, TPOSE>(p, buf, full, empty, stage_elems, \
                                                                                mfrag, stream0, rb, wg, lane);
    TSG_DMMA_RB(0) TSG_DMMA_RB(1) TSG_DMMA_RB(2) TSG_DMMA_RB(3) TSG_DMMA_RB(4) TSG_DMMA_RB(5) TSG_DMMA_RB(6)
    TSG_DMMA_RB(7)
#undef TSG_DMMA_RB
  } else {
    dmma_consumer<Real, KS, STAGES, std::conditional_t<SPARSE, DmmaRuntimeNz, DmmaDenseNz>, MREG, kDirectOut, -1, TPOSE>(
        p, buf, full, empty, stage_elems, mfrag, stream0, rb, wg, lane);
  }
}

template <typename Real, int KS, int STAGES, bool SPARSE, bool SIMT = false, bool TPOSE = false>
__global__ void __launch_bounds__(DShape<Real, KS>::kThreads + 32, DShape<Real, KS>::W >= 16 ? 1 : 2)
    k_stream_dmma(const __grid_constant__ DmmaParams<Real, KS> p) {
  k_stream_dmma_body<Real, KS, STAGES, SPARSE, SIMT, std::conditional_t<SPARSE, DmmaRuntimeNz, DmmaDenseNz>, TPOSE>(p);
}

// --------------------------------------------------------------------------
// k_dmma_direct: the same DMMA product without shared-memory staging of X.
// Every warp owns work items of 8*NR consecutive groups and runs them
// independently (no CTA barriers): it loads its B fragments straight from
// global memory (lane (lr, lc) reads element 4k+lc of group 8nb+lr: every
// 32-byte sector is fully used), multiplies by M fragments kept in shared
// memory in fragment order, and stores its C fragments back in place.  All
// loads of an item precede its stores, and items are disjoint, so the update
// is in-place safe.
template <int KS>
struct DdShape {
  static constexpr int D = 1 << KS;
  static constexpr int RB = D / 8;
  static constexpr int KST = D / 4;
  static constexpr int NR = KS >= 5 ? 1 : (KS == 4 ? 2 : 4);  // 8-group blocks per item
  static constexpr int GI = 8 * NR;                            // groups per item
  static constexpr int kWarps = 4;
};

template <int KS>
struct DdParams {
  double* re;
  double* im;
  const double* mat;  // [Mr | Mi | Ms], D x D each (device)
  uint64_t g_begin;
  uint64_t n_items;
  uint64_t fixed_or;
  uint64_t masks[kMaxMasks];
  int n_masks;
  uint64_t off[1 << KS];
  uint32_t nzblk[3];
};

template <int KS>
__device__ __forceinline__ uint64_t dd_base(const DdParams<KS>& p, uint64_t t) {
  uint64_t b = 0;
#pragma unroll
  for (int i = 0; i < kMaxMasks; ++i)
    if (i < p.n_masks) b += (t & p.masks[i]) << i;
  return b | p.fixed_or;
}

template <int KS, bool SPARSE>
__global__ void __launch_bounds__(32 * DdShape<KS>::kWarps) k_dmma_direct(const __grid_constant__ DdParams<KS> p) {
  using S = DdShape<KS>;
  __shared__ double mfrag[3 * S::KST * S::RB * 32];  // [m][k][rb][lane]
  {
    constexpr int DD = S::D * S::D;
    for (int f = threadIdx.x; f < 3 * S::KST * S::RB * 32; f += blockDim.x) {
      const int ln = f % 32, rbf = (f / 32) % S::RB, k = (f / (32 * S::RB)) % S::KST, m = f / (32 * S::RB * S::KST);
      mfrag[f] = p.mat[m * DD + (8 * rbf + (ln >> 2)) * S::D + 4 * k + (ln & 3)];
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  uint64_t offb[S::KST];
#pragma unroll
  for (int k = 0; k < S::KST; ++k) offb[k] = p.off[4 * k + lc];
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * S::kWarps;
  for (uint64_t item = static_cast<uint64_t>(blockIdx.x) * S::kWarps + warp; item < p.n_items; item += stride) {
    const uint64_t g0 = p.g_begin + item * S::GI;
    double xr[S::NR][S::KST], xi[S::NR][S::KST];
#pragma unroll
    for (int nb = 0; nb < S::NR; ++nb) {
      const uint64_t b = dd_base(p, g0 + 8 * nb + lr);
#pragma unroll
      for (int k = 0; k < S::KST; ++k) {
        xr[nb][k] = p.re[b + offb[k]];
        xi[nb][k] = p.im[b + offb[k]];
      }
    }
    double t1[S::RB][S::NR][2], t2[S::RB][S::NR][2], t3[S::RB][S::NR][2];
#pragma unroll
    for (int rb = 0; rb < S::RB; ++rb)
#pragma unroll
      for (int nb = 0; nb < S::NR; ++nb)
        t1[rb][nb][0] = t1[rb][nb][1] = t2[rb][nb][0] = t2[rb][nb][1] = t3[rb][nb][0] = t3[rb][nb][1] = 0.0;
#pragma unroll
    for (int k = 0; k < S::KST; ++k) {
#pragma unroll
      for (int rb = 0; rb < S::RB; ++rb) {
        const int bit = rb * S::KST + k;
        const double* mf = mfrag + (k * S::RB + rb) * 32 + lane;
        const double fr = mf[0], fi = mf[S::KST * S::RB * 32], fs = mf[2 * S::KST * S::RB * 32];
#pragma unroll
        for (int nb = 0; nb < S::NR; ++nb) {
          if (!SPARSE || ((p.nzblk[0] >> bit) & 1u)) dmma(t1[rb][nb], fr, xr[nb][k]);
          if (!SPARSE || ((p.nzblk[1] >> bit) & 1u)) dmma(t2[rb][nb], fi, xi[nb][k]);
          if (!SPARSE || ((p.nzblk[2] >> bit) & 1u)) dmma(t3[rb][nb], fs, xr[nb][k] + xi[nb][k]);
        }
      }
    }
#pragma unroll
    for (int nb = 0; nb < S::NR; ++nb)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint64_t b = dd_base(p, g0 + 8 * nb + 2 * lc + i);
#pragma unroll
        for (int rb = 0; rb < S::RB; ++rb) {
          const uint64_t a = b + p.off[8 * rb + lr];
          p.re[a] = t1[rb][nb][i] - t2[rb][nb][i];
          p.im[a] = t3[rb][nb][i] - t1[rb][nb][i] - t2[rb][nb][i];
        }
      }
  }
}

}  // namespace tsg
