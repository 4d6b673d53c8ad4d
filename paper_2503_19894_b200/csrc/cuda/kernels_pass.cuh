// k_pass: a run of fused gates applied in ONE streaming pass over HBM.
//
// Every gate in a fused circuit reads and writes the whole state once
// (2 * 2^n * B_amp bytes), so a circuit of G gates costs G HBM passes.  A
// pass kernel loads a tile of 2^M amplitudes into shared memory, applies a
// whole op list to it there, and writes it back once: G gates cost one pass
// plus their arithmetic.  Tiles are the 2^(M-L) runs of 2^L contiguous
// amplitudes selected by the pass's high tile qubits (PassLaunch::high): a
// warp moves two whole 256-byte runs per 16-byte-per-thread access.  Every
// consumer thread prefetches its share of tile j + STAGES - 1 with cp.async
// while the CTA works on tile j (STAGES tiles in flight per SM), and writes
// tile j back with 16-byte stores.  One bulk copy per run from a single
// producer warp could not keep up: ~1 TB/s chip-wide for 256-byte runs
// (profiles/r01 microbench: bulk-copy issue is ~300 cycles per thread).
//
// Ops (PassOp, gate_launch.hpp), in program order:
//   GEN   a non-diagonal sub-gate, block-diagonal in its "block" qubits
//         (tilesim::mixed_bits): the mixed qubits are tile qubits, the block
//         qubits (anywhere) select one 2^ks x 2^ks block per group.  One
//         thread per group: gather the 2^ks amplitudes from shared memory,
//         the dense row-by-column product with k_direct's FMA order (Zero
//         scalars are exact zeros of the snapped matrix), scatter in place.
//   RUN   a run of consecutive diagonal sub-gates (they commute; the host
//         orders them by class).  The amplitudes x = tid + i * kPassThreads
//         of a thread stay in registers for the whole run.  Table-index bits
//         outside the tile are per-tile constants (computed once per tile
//         for every op), DiagT ops (in-tile bits on thread-id positions only)
//         fold into one factor per thread, DiagI ops (in-tile bits on
//         iteration positions only) into one factor per iteration i shared
//         through shared memory, DiagX ops are applied amplitude by
//         amplitude.  Inactive controls select an identity entry appended to
//         every table (no divergent branches).
// The CTA synchronises with a barrier between ops that touch different
// amplitude sets.
#pragma once

#ifndef __CUDACC_RTC__  // NVRTC (pass_jit.cpp) supplies the integer types
#include <cstdint>
#include <type_traits>
#endif

#include "kernels_dmma.cuh"

namespace tsg {

// Loops whose trip counts come from op fields: fully unrolled in a JIT pass
// (the fields are constants there), left alone in the interpreter.
#ifdef TSG_JIT
#define TSG_JIT_UNROLL _Pragma("unroll")
#else
#define TSG_JIT_UNROLL
#endif

template <typename Real>
struct Real2Of;
template <>
struct Real2Of<double> {
  using T = double2;
};
template <>
struct Real2Of<float> {
  using T = float2;
};

struct PassParams {
  void* re;
  void* im;
  const unsigned char* blob;  // device copy, staged into shared memory
  int blob_bytes;             // multiple of 16
  int n_ops;
  uint64_t n_tiles;
  uint64_t tmask[kMaxMasks];  // tile id -> bits >= L (pre-shift), zeros at the high tile qubits
  int n_tmask;
};

template <typename Real, int M, int L>
struct PassShape {
  static constexpr int kRuns = 1 << (M - L);
  static constexpr int kRunLen = 1 << L;
  static constexpr int kStride = kRunLen + kPassPadBytes / static_cast<int>(sizeof(Real));
  static constexpr int kStageElems = kRuns * kStride;
  static constexpr int kIter = (1 << M) / kPassThreads;  // amplitudes per thread (register layout)
  static constexpr int kIterBits = M - kPassLogThreads;
  static_assert(kIter >= 1 && kIterBits <= 8, "tile / thread geometry");
  static constexpr size_t kFiBytes = 2 * kPassMaxGEntries * 2 * sizeof(Real);  // group tables, double-buffered
  static constexpr size_t kTcBytes = 2 * kPassMaxOps * sizeof(uint32_t);  // per-tile op constants, double-buffered
  static constexpr size_t smem_bytes(int blob_bytes, int stages) {
    return ((static_cast<size_t>(blob_bytes) + 127) & ~size_t{127}) +
           static_cast<size_t>(stages) * 2 * kStageElems * sizeof(Real) + kFiBytes + kTcBytes;
  }
};

__device__ __forceinline__ void consumer_bar() { __syncthreads(); }

// padded shared-memory offset of tile coordinate x
template <int L, int STRIDE>
__device__ __forceinline__ uint32_t pass_addr(uint32_t x) {
  return (x >> L) * STRIDE + (x & ((1u << L) - 1));
}

template <typename Real>
__device__ __forceinline__ void cmul_acc(Real& ar, Real& ai, Real br, Real bi) {
  const Real r = fma(ar, br, -ai * bi);
  ai = fma(ar, bi, ai * br);
  ar = r;
}

// --------------------------------------------------------------------- GEN
// Work item w = tid + kPassThreads * k: group g = w mod G' (G' = groups when
// groups >= kPassThreads), rows [R r, R r + R) with r = w / groups and
// R = D >> log2_rsplit.  With a row split every thread holds one item: all
// read their group, a consumer barrier, then all write (in place).
template <typename Real, int KS, int M, int L, int RSPLIT>
__device__ __forceinline__ void pass_gen(const PassOp& op, const unsigned char* blob, uint32_t jo, Real* xr,
                                         Real* xi, int tid) {
  using R2 = typename Real2Of<Real>::T;
  constexpr int D = 1 << KS;
  constexpr int R = D / RSPLIT;  // rows per item
  const unsigned char* data = blob + op.data_off;
  const uint32_t* soff_p = reinterpret_cast<const uint32_t*>(data);
  const uint32_t* et = reinterpret_cast<const uint32_t*>(data + ((4 * D + 15) & ~15));
  const uint32_t* ek = et + kPassThreads;
  const R2* blocks = reinterpret_cast<const R2*>(blob + op.aux_off);
  uint32_t soff[D];
#pragma unroll
  for (int j = 0; j < D; ++j) soff[j] = soff_p[j];
  const uint32_t n_groups = 1u << op.log2_groups;
  const uint32_t e0 = et[tid];
  const int r0 = RSPLIT > 1 ? (tid >> op.log2_groups) * R : 0;
  uint32_t k = 0;
  for (uint32_t g = tid; g < (RSPLIT > 1 ? uint32_t(kPassThreads) : n_groups); g += kPassThreads, ++k) {
    const uint32_t e = e0 + ek[k];
    const uint32_t a = e & 0xffffu;
    // blocks are D*D + 1 entries apart: lanes reading different blocks hit different banks
    const R2* mat = blocks + ((e >> 16) | jo) * (D * D + 1) + r0 * D;
    Real vr[D], vi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      vr[j] = xr[a + soff[j]];
      vi[j] = xi[a + soff[j]];
    }
    Real yr[R], yi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      yr[r] = Real(0);
      yi[r] = Real(0);
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const R2 m = mat[r * D + c];
        yr[r] = fma(m.x, vr[c], yr[r]);  // k_direct's order
        yi[r] = fma(m.x, vi[c], yi[r]);
        yr[r] = fma(-m.y, vi[c], yr[r]);
        yi[r] = fma(m.y, vr[c], yi[r]);
      }
      if constexpr (RSPLIT == 1) {
        xr[a + soff[r]] = yr[r];
        xi[a + soff[r]] = yi[r];
      }
    }
    if constexpr (RSPLIT > 1) {
      consumer_bar();  // every item of the tile has read its group
      if ((tid >> op.log2_groups) < RSPLIT) {  // threads without an item only join the barrier
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t so = soff_p[r0 + r];
          xr[a + so] = yr[r];
          xi[a + so] = yi[r];
        }
      }
    }
  }
}

// Perm: row r of the group takes element src[r] times val[r]; items as GEN
// (a row split gathers only the item's rows; a barrier separates the
// gathers from the in-place writes).
template <typename Real, int KS, int M, int L, int RSPLIT>
__device__ __forceinline__ void pass_perm(const PassOp& op, const unsigned char* blob, uint32_t jo, Real* xr,
                                          Real* xi, int tid) {
  using R2 = typename Real2Of<Real>::T;
  constexpr int D = 1 << KS;
  constexpr int R = D / RSPLIT;
  const unsigned char* data = blob + op.data_off;
  const uint32_t* soff_p = reinterpret_cast<const uint32_t*>(data);
  const uint32_t* et = reinterpret_cast<const uint32_t*>(data + ((4 * D + 15) & ~15));
  const uint32_t* ek = et + kPassThreads;
  constexpr int kSrcBytes = (4 * D + 15) & ~15;
  constexpr int kBlockBytes = kSrcBytes + D * static_cast<int>(sizeof(R2));
  const uint32_t n_groups = 1u << op.log2_groups;
  const uint32_t e0 = et[tid];
  const int r0 = RSPLIT > 1 ? (tid >> op.log2_groups) * R : 0;
  const bool active = RSPLIT == 1 || (tid >> op.log2_groups) < RSPLIT;
  uint32_t k = 0;
  for (uint32_t g = tid; g < (RSPLIT > 1 ? uint32_t(kPassThreads) : n_groups); g += kPassThreads, ++k) {
    const uint32_t e = e0 + ek[k];
    const uint32_t a = e & 0xffffu;
    const unsigned char* blk = blob + op.aux_off + ((e >> 16) | jo) * kBlockBytes;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(blk) + r0;
    const R2* val = reinterpret_cast<const R2*>(blk + kSrcBytes) + r0;
    Real vr[R], vi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t sa = a + src[r];
      vr[r] = xr[sa];
      vi[r] = xi[sa];
    }
    if constexpr (RSPLIT > 1) consumer_bar();  // every item has gathered before anyone writes
    if (active) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const R2 m = val[r];
        const Real yr = fma(-m.y, vi[r], m.x * vr[r]);  // k_direct's order for one nonzero entry
        const Real yi = fma(m.y, vr[r], m.x * vi[r]);
        const uint32_t so = soff_p[r0 + r];
        xr[a + so] = yr;
        xi[a + so] = yi;
      }
    }
  }
}

template <typename Real, int KS, int M, int L>
__device__ __forceinline__ void pass_perm_split(const PassOp& op, const unsigned char* blob, uint32_t jo, Real* xr,
                                                Real* xi, int tid) {
  constexpr int D = 1 << KS;
  switch (op.log2_rsplit) {  // see pass_gen_split
    case 0:
      if constexpr (KS <= 3 || (KS == 4 && sizeof(Real) == 4)) pass_perm<Real, KS, M, L, 1>(op, blob, jo, xr, xi, tid);
      break;
    case 1:
      if constexpr (D >= 2) pass_perm<Real, KS, M, L, 2>(op, blob, jo, xr, xi, tid);
      break;
    case 2:
      if constexpr (D >= 4) pass_perm<Real, KS, M, L, 4>(op, blob, jo, xr, xi, tid);
      break;
    default:
      if constexpr (D >= 8) pass_perm<Real, KS, M, L, 8>(op, blob, jo, xr, xi, tid);
      break;
  }
}

template <typename Real, int KS, int M, int L>
__device__ __forceinline__ void pass_gen_split(const PassOp& op, const unsigned char* blob, uint32_t jo, Real* xr,
                                               Real* xi, int tid) {
  constexpr int D = 1 << KS;
  // Without a row split only KS <= 3, or KS = 4 in complex64 (2^12-amplitude
  // tiles: 256 groups for 256 threads); complex128 tiles (2^11) always split KS >= 4.
  switch (op.log2_rsplit) {
    case 0:
      if constexpr (KS <= 3 || (KS == 4 && sizeof(Real) == 4)) pass_gen<Real, KS, M, L, 1>(op, blob, jo, xr, xi, tid);
      break;
    case 1:
      if constexpr (D >= 2) pass_gen<Real, KS, M, L, 2>(op, blob, jo, xr, xi, tid);
      break;
    case 2:
      if constexpr (D >= 4) pass_gen<Real, KS, M, L, 4>(op, blob, jo, xr, xi, tid);
      break;
    default:
      if constexpr (D >= 8) pass_gen<Real, KS, M, L, 8>(op, blob, jo, xr, xi, tid);
      break;
  }
}

template <typename Real, int M, int L>
__device__ __forceinline__ void pass_gen_dispatch(const PassOp& op, const unsigned char* blob, uint32_t jo, Real* xr,
                                                  Real* xi, int tid) {
  if (op.kind == kPassSPerm) {
    switch (op.ks) {
      case 1: pass_perm_split<Real, 1, M, L>(op, blob, jo, xr, xi, tid); break;
      case 2: pass_perm_split<Real, 2, M, L>(op, blob, jo, xr, xi, tid); break;
      case 3: pass_perm_split<Real, 3, M, L>(op, blob, jo, xr, xi, tid); break;
      case 4: pass_perm_split<Real, 4, M, L>(op, blob, jo, xr, xi, tid); break;
      default: pass_perm_split<Real, 5, M, L>(op, blob, jo, xr, xi, tid); break;
    }
    return;
  }
  switch (op.ks) {
    case 1: pass_gen_split<Real, 1, M, L>(op, blob, jo, xr, xi, tid); break;
    case 2: pass_gen_split<Real, 2, M, L>(op, blob, jo, xr, xi, tid); break;
    case 3: pass_gen_split<Real, 3, M, L>(op, blob, jo, xr, xi, tid); break;
    case 4: pass_gen_split<Real, 4, M, L>(op, blob, jo, xr, xi, tid); break;
    default:
      if constexpr (sizeof(Real) == 4) {
        if (op.ks == 5) pass_gen_split<Real, 5, M, L>(op, blob, jo, xr, xi, tid);
      }
      break;
  }
}

// ---------------------------------------------------------- register ops
// compile-time deposit of the bits of j into the set bits of mask
__host__ __device__ constexpr int deposit_c(int j, int mask) {
  int out = 0;
  for (int b = 0, k = 0; b < 8; ++b)
    if ((mask >> b) & 1) out |= ((j >> k++) & 1) << b;
  return out;
}

// RGen / RPerm on the thread's R registers: the op mixes register bits RM;
// sub-group s (register index with the RM bits clear) uses block
// tc | thread-position block bits | register block bits of s.
template <typename Real, int R, int RM, bool PERM>
__device__ __forceinline__ void reg_gen(const PassOp& op, const unsigned char* blob, uint32_t tc, int tid,
                                        Real (&ar)[R], Real (&ai)[R]) {
  using R2 = typename Real2Of<Real>::T;
  constexpr int KE = cx_popc(RM);
  constexpr int D = 1 << KE;
  uint32_t jt = tc;
  const int thr_off = op.thr_off;
  if (thr_off >= 0) {  // host table: block bits on thread positions; 0xff = controls inactive
    const uint32_t v = blob[thr_off + tid];
    if (v == 0xffu) return;
    jt |= v;
  }
  // the op's register-bit fields, once (the sub-group loop below is unrolled)
  constexpr int kRegBits = cx_ctz(R);
  uint32_t dep[kRegBits > 0 ? kRegBits : 1];
#pragma unroll
  for (int k = 0; k < kRegBits; ++k) dep[k] = op.dep[k];
  const uint32_t ictl_mask = op.ictl_mask, ictl_val = op.ictl_val;
  const unsigned char* blocks = blob + op.aux_off;
  constexpr int kSrcBytes = (4 * D + 15) & ~15;
  constexpr int kBlockBytes = PERM ? kSrcBytes + D * static_cast<int>(sizeof(R2)) : (D * D + 1) * static_cast<int>(sizeof(R2));
  if constexpr (!PERM && R / D > 1) {
    // every sub-group uses the same block (no block bits on register
    // positions, no register controls): each matrix entry is read once and
    // applied to all R / D sub-groups, with each output's FMA sequence (and
    // so its rounding) unchanged
    bool uniform = ictl_mask == 0;
#pragma unroll
    for (int k = 0; k < kRegBits; ++k) uniform = uniform && (((RM >> k) & 1) || dep[k] == 0);
    if (uniform) {
      constexpr int NS = R / D;
      const R2* mat = reinterpret_cast<const R2*>(blocks + jt * kBlockBytes);
      Real vr[NS][D], vi[NS][D];
#pragma unroll
      for (int q = 0, s = 0; s < R; ++s) {
        if (s & RM) continue;  // compile time
#pragma unroll
        for (int j = 0; j < D; ++j) {
          vr[q][j] = ar[s | deposit_c(j, RM)];
          vi[q][j] = ai[s | deposit_c(j, RM)];
        }
        ++q;
      }
#pragma unroll
      for (int r = 0; r < D; ++r) {
        Real yr[NS], yi[NS];
#pragma unroll
        for (int q = 0; q < NS; ++q) yr[q] = yi[q] = Real(0);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const R2 m = mat[r * D + c];
#pragma unroll
          for (int q = 0; q < NS; ++q) {
            yr[q] = fma(m.x, vr[q][c], yr[q]);  // k_direct's order
            yi[q] = fma(m.x, vi[q][c], yi[q]);
            yr[q] = fma(-m.y, vi[q][c], yr[q]);
            yi[q] = fma(m.y, vr[q][c], yi[q]);
          }
        }
#pragma unroll
        for (int q = 0, s = 0; s < R; ++s) {
          if (s & RM) continue;
          ar[s | deposit_c(r, RM)] = yr[q];
          ai[s | deposit_c(r, RM)] = yi[q];
          ++q;
        }
      }
      return;
    }
  }
#pragma unroll
  for (int s = 0; s < R; ++s) {
    if (s & RM) continue;  // compile time
    if ((static_cast<uint32_t>(s) & ictl_mask) != ictl_val) continue;
    uint32_t jb = jt;
#pragma unroll
    for (int k = 0; k < kRegBits; ++k)
      if ((s >> k) & 1) jb |= dep[k];
    const unsigned char* blk = blocks + jb * kBlockBytes;
    Real vr[D], vi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      vr[j] = ar[s | deposit_c(j, RM)];
      vi[j] = ai[s | deposit_c(j, RM)];
    }
    if constexpr (PERM) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(blk);
      const R2* val = reinterpret_cast<const R2*>(blk + kSrcBytes);
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const uint32_t c = src[r];
        Real xr = vr[0], xi = vi[0];
#pragma unroll
        for (int q = 1; q < D; ++q)
          if (c == static_cast<uint32_t>(q)) {
            xr = vr[q];
            xi = vi[q];
          }
        const R2 m = val[r];
        ar[s | deposit_c(r, RM)] = fma(-m.y, xi, m.x * xr);  // k_direct's order for one nonzero entry
        ai[s | deposit_c(r, RM)] = fma(m.y, xr, m.x * xi);
      }
    } else {
      const R2* mat = reinterpret_cast<const R2*>(blk);
#pragma unroll
      for (int r = 0; r < D; ++r) {
        Real yr = Real(0), yi = Real(0);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const R2 m = mat[r * D + c];
          yr = fma(m.x, vr[c], yr);  // k_direct's order
          yi = fma(m.x, vi[c], yi);
          yr = fma(-m.y, vi[c], yr);
          yi = fma(m.y, vr[c], yi);
        }
        ar[s | deposit_c(r, RM)] = yr;
        ai[s | deposit_c(r, RM)] = yi;
      }
    }
  }
}

// rmask: mixed bits among the r register bits (at most 3 of them)
template <typename Real, int R, bool PERM, int RM = 1>
__device__ __forceinline__ void reg_gen_dispatch(const PassOp& op, const unsigned char* blob, uint32_t tc, int tid,
                                                 Real (&ar)[R], Real (&ai)[R]) {
  if constexpr (RM < R) {
    if constexpr (cx_popc(RM) <= 3) {
      if (op.rmask == RM) {
        reg_gen<Real, R, RM, PERM>(op, blob, tc, tid, ar, ai);
        return;
      }
    }
    reg_gen_dispatch<Real, R, PERM, RM + 1>(op, blob, tc, tid, ar, ai);
  }
}

// --------------------------------------------------------------------- RUN
template <typename Real>
__device__ __forceinline__ typename Real2Of<Real>::T diag_entry(const PassOp& op, const unsigned char* blob,
                                                                 uint32_t j) {
  return reinterpret_cast<const typename Real2Of<Real>::T*>(blob + op.data_off)[j];
}

// The RUN header at ops[o] (ks = groups, log2_groups = per-op DiagT count,
// log2_rsplit = per-op DiagX count) is followed by its groups (a DGroup
// header and its DMember ops each), then the per-op DiagT and DiagX ops.
// Groups: every thread builds some entries of the groups' combined tables
// (product of the members' factors at that signature index), a barrier,
// then every amplitude multiplies one entry per group.  Returns the op after
// the run.  gtab: this run's table scratch (kPassMaxGEntries entries).
template <typename Real, int R>
__device__ __forceinline__ int pass_diag_run(const PassOp* ops, int o, const unsigned char* blob, const uint32_t* tcs,
                                             int tid, Real (&ar)[R], Real (&ai)[R], typename Real2Of<Real>::T* gtab) {
  using R2 = typename Real2Of<Real>::T;
  constexpr int kBits = cx_ctz(R);
  const int n_groups = ops[o].ks, nT = ops[o].log2_groups, nX = ops[o].log2_rsplit;
  ++o;
  if (n_groups > 0) {
    // build: entry e of group g = product over members (inactive controls
    // skip); the groups' entries are laid out back to back in gtab (at most
    // kPassMaxGEntries <= kPassThreads), so thread tid builds flat entry tid:
    // every group in parallel, one short member chain per thread
    static_assert(kPassMaxGEntries <= kPassThreads, "one group entry per thread");
    int og = o;
    TSG_JIT_UNROLL
    for (int g = 0; g < n_groups; ++g) {
      const PassOp& gh = ops[og];
      const int sbits = gh.ks, m = gh.log2_groups;
      const int e = tid - gh.data_off;
      if (e >= 0 && e < (1 << sbits)) {
        // two interleaved partial products halve the dependent multiply chain
        Real fr[2] = {Real(1), Real(1)}, fi[2] = {Real(0), Real(0)};
        TSG_JIT_UNROLL
        for (int t = 1; t <= m; ++t) {
          const PassOp& mo = ops[og + t];
          const uint32_t tc = tcs[og + t];
          if (tc == ~0u || (static_cast<uint32_t>(e) & mo.ictl_mask) != mo.ictl_val) continue;
          uint32_t jj = tc;
#pragma unroll
          for (int k = 0; k < kPassMaxSig; ++k)
            if (((e >> k) & 1) && k < sbits) jj |= mo.dep[k];
          const R2 d = diag_entry<Real>(mo, blob, jj);
          cmul_acc(fr[t & 1], fi[t & 1], d.x, d.y);
        }
        cmul_acc(fr[0], fi[0], fr[1], fi[1]);
        gtab[gh.data_off + e] = R2{fr[0], fi[0]};
      }
      og += 1 + m;
    }
    consumer_bar();
    // apply: one entry per group and amplitude
    og = o;
    TSG_JIT_UNROLL
    for (int g = 0; g < n_groups; ++g) {
      const PassOp& gh = ops[og];
      const uint32_t tv = blob[gh.aux_off + tid];
      uint32_t dep[kBits > 0 ? kBits : 1];
#pragma unroll
      for (int k = 0; k < kBits; ++k) dep[k] = gh.dep[k];
      const R2* gt = gtab + gh.data_off;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        uint32_t idx = tv;
#pragma unroll
        for (int k = 0; k < kBits; ++k)
          if ((i >> k) & 1) idx |= dep[k];
        const R2 f = gt[idx];
        cmul_acc(ar[i], ai[i], f.x, f.y);
      }
      og += 1 + gh.log2_groups;
    }
    o = og;
  }
  // DiagT: one factor per thread (two interleaved partial products)
  Real ftr = Real(1), fti = Real(0), f2r = Real(1), f2i = Real(0);
  int t = 0;
  TSG_JIT_UNROLL
  for (; t + 1 < nT; t += 2) {
    const PassOp& op0 = ops[o + t];
    const PassOp& op1 = ops[o + t + 1];
    // inactive (tc = ~0 or tv = 0xff) selects the identity entry 2^ks (<= 128)
    const R2 d0 = diag_entry<Real>(op0, blob, min(tcs[o + t] | blob[op0.aux_off + tid], 1u << op0.ks));
    const R2 d1 = diag_entry<Real>(op1, blob, min(tcs[o + t + 1] | blob[op1.aux_off + tid], 1u << op1.ks));
    cmul_acc(ftr, fti, d0.x, d0.y);
    cmul_acc(f2r, f2i, d1.x, d1.y);
  }
  if (t < nT) {
    const PassOp& op = ops[o + t];
    const R2 d = diag_entry<Real>(op, blob, min(tcs[o + t] | blob[op.aux_off + tid], 1u << op.ks));
    cmul_acc(ftr, fti, d.x, d.y);
  }
  if (nT > 0) {
    if (nT > 1) cmul_acc(ftr, fti, f2r, f2i);
#pragma unroll
    for (int i = 0; i < R; ++i) cmul_acc(ar[i], ai[i], ftr, fti);
  }
  o += nT;
  // DiagX: amplitude by amplitude, k_diag's update
  TSG_JIT_UNROLL
  for (int x = 0; x < nX; ++x, ++o) {
    const PassOp& op = ops[o];
    const uint32_t tc = tcs[o];
    const uint32_t tv = blob[op.aux_off + tid];
    if ((tc >> 31) || tv == 0xffu) continue;
    const uint32_t jc = tc | tv;
    uint32_t dep[kBits > 0 ? kBits : 1];
#pragma unroll
    for (int k = 0; k < kBits; ++k) dep[k] = op.dep[k];
    const uint32_t im = op.ictl_mask, iv = op.ictl_val, one = 1u << op.ks;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      uint32_t j = jc;
#pragma unroll
      for (int k = 0; k < kBits; ++k)
        if ((i >> k) & 1) j |= dep[k];
      const R2 d = diag_entry<Real>(op, blob, (static_cast<uint32_t>(i) & im) == iv ? j : one);
      const Real r0 = ar[i], i0 = ai[i];
      ar[i] = fma(d.x, r0, -d.y * i0);
      ai[i] = fma(d.x, i0, d.y * r0);
    }
  }
  return o;
}

// ------------------------------------------------------------------ kernel
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Tile transfers: 16-byte chunks, chunk c of array (c / kChunksPerArray) at
// element (c % kChunksPerArray) * kEpc of the tile's run-major order; every
// consumer thread moves kChunks / kPassThreads chunks (a warp covers 512
// contiguous bytes = two 256-byte runs).
template <typename Real, int M, int L>
struct PassCopy {
  using S = PassShape<Real, M, L>;
  static constexpr int kEpc = 16 / sizeof(Real);                   // elements per 16-byte chunk
  static constexpr int kChunksPerArray = (1 << M) / kEpc;
  static constexpr int kPerThread = 2 * kChunksPerArray / kPassThreads;
  static_assert(kPerThread >= 1 && (2 * kChunksPerArray) % kPassThreads == 0, "copy split");
  static_assert(S::kRunLen % kEpc == 0, "runs are whole chunks");
};

// Registers <-> tile in shared memory.  When the layout's lowest register
// positions are the tile's lowest positions (vb of them), the registers
// i .. i + 2^vb - 1 are consecutive elements of one 16-byte unit: one vector
// access each (complex64: a warp then moves whole 16-byte units instead of
// piling 4-byte accesses onto a few banks; complex128 keeps scalar moves).
template <typename Real, int R>
__device__ __forceinline__ void regs_to_smem(Real* xr, Real* xi, const uint32_t (&at)[R], const Real (&ar)[R],
                                             const Real (&ai)[R], int vb) {
  if constexpr (sizeof(Real) == 4 && R % 4 == 0) {
    if (vb >= 2) {
#pragma unroll
      for (int i = 0; i < R; i += 4) {
        *reinterpret_cast<float4*>(xr + at[i]) = make_float4(ar[i], ar[i + 1], ar[i + 2], ar[i + 3]);
        *reinterpret_cast<float4*>(xi + at[i]) = make_float4(ai[i], ai[i + 1], ai[i + 2], ai[i + 3]);
      }
      return;
    }
  }
  if constexpr (sizeof(Real) == 4 && R % 2 == 0) {
    if (vb >= 1) {
      using V2 = float2;
#pragma unroll
      for (int i = 0; i < R; i += 2) {
        *reinterpret_cast<V2*>(xr + at[i]) = V2{ar[i], ar[i + 1]};
        *reinterpret_cast<V2*>(xi + at[i]) = V2{ai[i], ai[i + 1]};
      }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    xr[at[i]] = ar[i];
    xi[at[i]] = ai[i];
  }
}

template <typename Real, int R>
__device__ __forceinline__ void smem_to_regs(const Real* xr, const Real* xi, const uint32_t (&at)[R], Real (&ar)[R],
                                             Real (&ai)[R], int vb) {
  if constexpr (sizeof(Real) == 4 && R % 4 == 0) {
    if (vb >= 2) {
#pragma unroll
      for (int i = 0; i < R; i += 4) {
        const float4 a = *reinterpret_cast<const float4*>(xr + at[i]);
        const float4 b = *reinterpret_cast<const float4*>(xi + at[i]);
        ar[i] = a.x, ar[i + 1] = a.y, ar[i + 2] = a.z, ar[i + 3] = a.w;
        ai[i] = b.x, ai[i + 1] = b.y, ai[i + 2] = b.z, ai[i + 3] = b.w;
      }
      return;
    }
  }
  if constexpr (sizeof(Real) == 4 && R % 2 == 0) {
    if (vb >= 1) {
      using V2 = float2;
#pragma unroll
      for (int i = 0; i < R; i += 2) {
        const V2 a = *reinterpret_cast<const V2*>(xr + at[i]);
        const V2 b = *reinterpret_cast<const V2*>(xi + at[i]);
        ar[i] = a.x, ar[i + 1] = a.y;
        ai[i] = b.x, ai[i + 1] = b.y;
      }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    ar[i] = xr[at[i]];
    ai[i] = xi[at[i]];
  }
}

// Layout change in registers: register bit K trades places with lane bit l
// (warp shuffles, no shared memory, no barrier).  For each register pair
// {i, i | 2^K} a thread keeps the element whose bit K equals its own lane
// bit; the other one comes from its partner lane (lane ^ 2^l), which sends
// its element with bit K equal to the receiver's lane bit: one shuffle per
// pair and array, the data moved unchanged (bit-identical to the
// shared-memory change).
template <int K, typename Real, int R>
__device__ __forceinline__ void shfl_swap_bit(Real (&ar)[R], Real (&ai)[R], int l, int lane) {
  const bool lb = (lane >> l) & 1;
  const int mask = 1 << l;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    if (i & (1 << K)) continue;  // compile time
    const int j = i | (1 << K);
    const Real sr = lb ? ar[i] : ar[j], si = lb ? ai[i] : ai[j];
    const Real rr = __shfl_xor_sync(0xffffffffu, sr, mask), ri = __shfl_xor_sync(0xffffffffu, si, mask);
    if (lb) {
      ar[i] = rr;
      ai[i] = ri;
    } else {
      ar[j] = rr;
      ai[j] = ri;
    }
  }
}

template <typename Real, int R>
__device__ __forceinline__ void shfl_swap(Real (&ar)[R], Real (&ai)[R], int k, int l, int lane) {
  constexpr int kBits = cx_ctz(R);
  if constexpr (kBits > 0) if (k == 0) return shfl_swap_bit<0>(ar, ai, l, lane);
  if constexpr (kBits > 1) if (k == 1) return shfl_swap_bit<1>(ar, ai, l, lane);
  if constexpr (kBits > 2) if (k == 2) return shfl_swap_bit<2>(ar, ai, l, lane);
  if constexpr (kBits > 3) if (k == 3) return shfl_swap_bit<3>(ar, ai, l, lane);
}

// Per-thread interpreter state of one tile: the registers of the current
// layout, their shared-memory offsets, and what carries across ops.
template <typename Real, int R>
struct PassRegs {
  Real ar[R], ai[R];
  uint32_t at[R];    // padded shared-memory offsets of the registers (current layout)
  int vb = 0;        // vector width (log2) of the current layout's register <-> smem moves
  uint32_t xt = 0;   // tile coordinate of the thread part of the current layout
  uint32_t irun = 0; // runs with diagonal groups so far (table double-buffering)
  bool in_smem = true;  // the registers have been stored (shared memory is current)
};

// One op (or one RUN with its members) of a tile; returns the next op index.
// The interpreter calls it in a loop over the blob's op table; a JIT-compiled
// pass (pass_jit.cpp) calls it once per op with `ops` a constexpr table and
// `o` a literal, so every field folds to a constant.
template <typename Real, int M, int L>
__device__ __forceinline__ int pass_step(const PassOp* ops, int o, int n_ops, const unsigned char* blob,
                                         const uint32_t* tcs, int tid, Real* xr, Real* xi,
                                         typename Real2Of<Real>::T* fi_tab,
                                         PassRegs<Real, PassShape<Real, M, L>::kIter>& rg) {
  using S = PassShape<Real, M, L>;
  constexpr int R = S::kIter;
  const PassOp& op = ops[o];
  const int kind = op.kind;
  if (kind == kPassLayout) {
    if (op.n_swap > 0 && !rg.in_smem) {
      // register <-> lane bit swaps within each warp; the new layout's
      // shared-memory offsets (for a later store) from its table as below
      TSG_JIT_UNROLL
      for (int q = 0; q < op.n_swap; ++q) shfl_swap<Real, R>(rg.ar, rg.ai, op.swap_k[q], op.swap_l[q], tid & 31);
    } else if (!rg.in_smem) {
      regs_to_smem<Real, R>(xr, xi, rg.at, rg.ar, rg.ai, rg.vb);
      consumer_bar();  // the tile is in shared memory in full
    } else if (o > 0) {
      consumer_bar();  // after shared-memory ops: their writes are visible
    }
    rg.xt = reinterpret_cast<const uint32_t*>(blob + op.aux_off)[tid];  // host-built per-thread coordinate
    const uint32_t at0 = pass_addr<L, S::kStride>(rg.xt);
    constexpr int kBits = cx_ctz(R);
    uint32_t pd[kBits];  // padded offset of each register position (additive over disjoint bits)
#pragma unroll
    for (int k = 0; k < kBits; ++k) pd[k] = op.dep[k];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      uint32_t a = at0;
#pragma unroll
      for (int k = 0; k < kBits; ++k)
        if ((i >> k) & 1) a += pd[k];
      rg.at[i] = a;
    }
    rg.vb = op.ks;  // vector width of this layout (host: lowest register positions = lowest tile positions)
    if (op.n_swap == 0 || rg.in_smem) smem_to_regs<Real, R>(xr, xi, rg.at, rg.ar, rg.ai, rg.vb);
    rg.in_smem = false;
    return o + 1;
  }
  if (kind == kPassRun) {
    // group tables alternate buffers run by run (each such run has a barrier)
    const bool has_groups = op.ks > 0;
    o = pass_diag_run<Real, R>(ops, o, blob, tcs, tid, rg.ar, rg.ai, fi_tab + (rg.irun & 1) * kPassMaxGEntries);
    rg.irun += has_groups;
    return o;
  }
  if (kind == kPassRGen || kind == kPassRPerm) {
    const uint32_t tc = tcs[o];
    if (!(tc >> 31)) {
      if (kind == kPassRPerm) reg_gen_dispatch<Real, R, true>(op, blob, tc, tid, rg.ar, rg.ai);
      else reg_gen_dispatch<Real, R, false>(op, blob, tc, tid, rg.ar, rg.ai);
    }
    return o + 1;
  }
  // SGen / SPerm: through shared memory
  if (!rg.in_smem) {
    regs_to_smem<Real, R>(xr, xi, rg.at, rg.ar, rg.ai, rg.vb);
    rg.in_smem = true;
  }
  consumer_bar();
  // the skip is tile-uniform, so a row-split op's internal barrier stays uniform
  const uint32_t tc = tcs[o];
  if (!(tc >> 31)) pass_gen_dispatch<Real, M, L>(op, blob, tc, xr, xi, tid);
  ++o;
  if (o < n_ops && ops[o].kind != kPassSGen && ops[o].kind != kPassSPerm && ops[o].kind != kPassLayout) {
    consumer_bar();  // back to the registers of the current layout
    smem_to_regs<Real, R>(xr, xi, rg.at, rg.ar, rg.ai, rg.vb);
    rg.in_smem = false;
  }
  return o;
}

// Op interpreter over the blob's op table (the generic k_pass).
struct PassInterp {
  template <typename Real, int M, int L, typename RG>
  static __device__ __forceinline__ void run(const PassOp* ops, int n_ops, const unsigned char* blob,
                                             const uint32_t* tcs, int tid, Real* xr, Real* xi,
                                             typename Real2Of<Real>::T* fi_tab, RG& rg) {
    for (int o = 0; o < n_ops;) o = pass_step<Real, M, L>(ops, o, n_ops, blob, tcs, tid, xr, xi, fi_tab, rg);
  }
};

// The tile pipeline; EXEC applies the op list to a tile (PassInterp, or a
// generated straight-line sequence in a JIT-compiled pass).
template <typename Real, int M, int L, int STAGES, typename EXEC>
__device__ __forceinline__ void k_pass_body(const PassParams& p) {
  using S = PassShape<Real, M, L>;
  using C = PassCopy<Real, M, L>;
  using R2 = typename Real2Of<Real>::T;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* blob = smem_raw;
  const int blob_round = (p.blob_bytes + 127) & ~127;
  Real* buf = reinterpret_cast<Real*>(smem_raw + blob_round);  // [STAGES][2][kStageElems]
  R2* fi_tab = reinterpret_cast<R2*>(reinterpret_cast<unsigned char*>(buf) + sizeof(Real) * 2 * STAGES * S::kStageElems);
  uint32_t* tc_tab = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(fi_tab) + S::kFiBytes);
  Real* gre = static_cast<Real*>(p.re);
  Real* gim = static_cast<Real*>(p.im);
  const int tid = threadIdx.x;

  {  // stage the blob (16-byte vectors)
    const uint4* src = reinterpret_cast<const uint4*>(p.blob);
    uint4* dst = reinterpret_cast<uint4*>(blob);
    for (int i = tid; i < p.blob_bytes / 16; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const uint64_t* roff = reinterpret_cast<const uint64_t*>(blob);
  const PassOp* ops = reinterpret_cast<const PassOp*>(blob + S::kRuns * sizeof(uint64_t));

  auto tile_base = [&](uint64_t tile) {
    uint64_t b = 0;
#pragma unroll
    for (int i = 0; i < kMaxMasks; ++i)
      if (i < p.n_tmask) b += (tile & p.tmask[i]) << i;
    return b << L;
  };
  // this thread's chunks: array, global element offset within the tile, stage offset
  Real* c_arr[C::kPerThread];
  uint64_t c_gofs[C::kPerThread];
  uint32_t c_off[C::kPerThread];
#pragma unroll
  for (int q = 0; q < C::kPerThread; ++q) {
    const int c = tid + q * kPassThreads;
    const int arr = c / C::kChunksPerArray;
    const int e = (c % C::kChunksPerArray) * C::kEpc;
    c_arr[q] = arr ? gim : gre;
    c_gofs[q] = roff[e >> L] + (e & (S::kRunLen - 1));
    c_off[q] = static_cast<uint32_t>(arr * S::kStageElems + (e >> L) * S::kStride + (e & (S::kRunLen - 1)));
  }
  const uint64_t first = blockIdx.x, step = gridDim.x;
  // Tile bases of the prefetch stream, stepped in the masked domain: with
  // the non-tile bits forced to 1, adding deposit(step) carries across them
  // (pdep(t + s) = ((pdep(t) | ~mask) + pdep(s)) & mask).
  const uint64_t tmask_all = tile_base(p.n_tiles - 1);  // every tile-id bit position
  const uint64_t dstep = tile_base(step);
  uint64_t pbase = tile_base(first);
  // bases of the tiles in flight (ring, oldest first)
  uint64_t ring[STAGES];
  uint64_t ptile = first;
  auto prefetch = [&](int s) {
#pragma unroll
    for (int r = 0; r + 1 < STAGES; ++r) ring[r] = ring[r + 1];
    if (ptile < p.n_tiles) {
      ring[STAGES - 1] = pbase;
      Real* st = buf + (2 * s) * S::kStageElems;
#pragma unroll
      for (int q = 0; q < C::kPerThread; ++q) cp_async16(st + c_off[q], c_arr[q] + pbase + c_gofs[q]);
    }
    cp_async_commit();  // one group per tile slot, empty past the end
    ptile += step;
    pbase = ((pbase | ~tmask_all) + dstep) & tmask_all;
  };
#pragma unroll
  for (int s = 0; s < STAGES; ++s) ring[s] = 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) prefetch(s);

  constexpr int R = S::kIter;  // amplitudes per thread (register layout)
  PassRegs<Real, R> rg;
  uint32_t j = 0;
  for (uint64_t tile = first; tile < p.n_tiles; tile += step, ++j) {
    const int s = static_cast<int>(j % STAGES);
    const uint64_t tbase = ring[1];  // tile j (ring[1..] = tiles j .. j + STAGES - 2 before this prefetch)
    // Tile-uniform op constants: table / block index bits outside the tile;
    // all ones when the controls outside the tile are inactive.  Double-buffered by tile
    // parity (a thread writing tile j + 2's buffer has passed tile j + 1's
    // first barrier, so nobody reads tile j's any more).
    uint32_t* tcs = tc_tab + (j & 1) * kPassMaxOps;
    for (int o = tid; o < p.n_ops; o += kPassThreads) {
      const PassOp& op = ops[o];
      uint32_t v = 0;
      for (int b = 0; b < op.n_out; ++b) v |= static_cast<uint32_t>((tbase >> op.out_gbit[b]) & 1u) << op.out_jbit[b];
      tcs[o] = (tbase & op.cout_mask) != op.cout_val ? ~0u : v;
    }
    cp_async_wait<STAGES - 2>();  // this thread's chunks of tile j have landed
    consumer_bar();               // ... and everyone's; the stage of tile j - 1 is stored
    prefetch(static_cast<int>((j + STAGES - 1) % STAGES));
    Real* xr = buf + (2 * s) * S::kStageElems;
    Real* xi = xr + S::kStageElems;
    // The op list starts with a LAYOUT op; registers hold the tile from then on.
    rg.in_smem = true;
    EXEC::template run<Real, M, L>(ops, p.n_ops, blob, tcs, tid, xr, xi, fi_tab, rg);
    if (!rg.in_smem) regs_to_smem<Real, R>(xr, xi, rg.at, rg.ar, rg.ai, rg.vb);
    consumer_bar();  // all ops done: write the tile back
    const Real* st = buf + (2 * s) * S::kStageElems;
#pragma unroll
    for (int q = 0; q < C::kPerThread; ++q)
      *reinterpret_cast<uint4*>(c_arr[q] + tbase + c_gofs[q]) = *reinterpret_cast<const uint4*>(st + c_off[q]);
  }
  cp_async_wait<0>();
}

template <typename Real, int M, int L, int STAGES>
__global__ void __launch_bounds__(kPassThreads, 2) k_pass(const __grid_constant__ PassParams p) {
  k_pass_body<Real, M, L, STAGES, PassInterp>(p);
}

}  // namespace tsg
