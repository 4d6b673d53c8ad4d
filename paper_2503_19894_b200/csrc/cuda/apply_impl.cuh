// Launch-side dispatch for one precision: GateLaunch -> kernel template
// instance + grid.  Included once per precision (apply_f64.cu, apply_f32.cu)
// so the two halves of the instantiation set compile in parallel.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <cstdlib>
#include <string>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.cuh"
#include "kernels_dmma.cuh"
#include "kernels_stream.cuh"
#include "kernels_umma.cuh"

#ifndef TSG_UMMA_DEFAULT_KS
#define TSG_UMMA_DEFAULT_KS 0x70u  // ks 4, 5, 6
#endif

namespace tsg {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

template <typename Real>
struct PrecisionTraits;
template <>
struct PrecisionTraits<double> {
  static constexpr int kDirectMax = 4;  // dense ks=5 c128 is FP64-bound: tile
  static constexpr int kMaxV = 2;       // 16-byte vectors
};
template <>
struct PrecisionTraits<float> {
  static constexpr int kDirectMax = 5;
  static constexpr int kMaxV = 4;
};

inline int lowest_target_bit(const GateLaunch& g) {
  // masks[0] covers t bits below the lowest target: its popcount is that position
  return g.n_masks > 0 ? __builtin_popcountll(g.masks[0]) : 64;
}

inline unsigned grid_for(uint64_t work, int num_sms, int per_sm = 32) {
  const uint64_t blocks = (work + 255) / 256;
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(blocks, uint64_t(num_sms) * per_sm)));
}

// ----------------------------------------------------------------- direct
template <typename Real, int KS, int V, bool SP>
void run_direct(const GateLaunch& g, cudaStream_t s, int num_sms) {
  DirectParams<Real, KS> p;
  std::memset(&p, 0, sizeof p);
  constexpr int D = 1 << KS;
  p.re = static_cast<Real*>(g.re);
  p.im = static_cast<Real*>(g.im);
  p.g_begin = g.g_begin;
  p.n_work = (g.g_end - g.g_begin) / V;
  p.fixed_or = g.fixed_or;
  p.n_masks = g.n_masks;
  for (int i = 0; i < g.n_masks; ++i) p.masks[i] = g.masks[i];
  for (int j = 0; j < D; ++j) p.off[j] = g.off[j];
  for (int e = 0; e < D * D; ++e) {
    p.mre[e] = static_cast<Real>(g.m_re[e]);
    p.mim[e] = static_cast<Real>(g.m_im[e]);
    if (g.m_re[e] != 0.0) p.nz[(2 * e) >> 5] |= 1u << ((2 * e) & 31);
    if (g.m_im[e] != 0.0) p.nz[(2 * e + 1) >> 5] |= 1u << ((2 * e + 1) & 31);
  }
  if (p.n_work == 0) return;
  k_direct<Real, KS, V, SP><<<static_cast<unsigned>((p.n_work + 255) / 256), 256, 0, s>>>(p);
  cuda_check(cudaGetLastError(), "k_direct launch");
}

template <typename Real, int KS>
void pick_direct(const GateLaunch& g, cudaStream_t s, int num_sms) {
  constexpr int VC = DirectShape<Real, KS>::kVCap;
  const uint64_t count = g.g_end - g.g_begin;
  const int low = lowest_target_bit(g);  // consecutive groups are adjacent below it
  auto fits = [&](int v, int log2v) { return VC >= v && low >= log2v && g.g_begin % v == 0 && count % v == 0; };
  if constexpr (VC >= 4) {
    if (fits(4, 2)) {
      g.sparse ? run_direct<Real, KS, 4, true>(g, s, num_sms) : run_direct<Real, KS, 4, false>(g, s, num_sms);
      return;
    }
  }
  if constexpr (VC >= 2) {
    if (fits(2, 1)) {
      g.sparse ? run_direct<Real, KS, 2, true>(g, s, num_sms) : run_direct<Real, KS, 2, false>(g, s, num_sms);
      return;
    }
  }
  g.sparse ? run_direct<Real, KS, 1, true>(g, s, num_sms) : run_direct<Real, KS, 1, false>(g, s, num_sms);
}

// ------------------------------------------------------------------- diag
template <typename Real, int KD, int V>
void run_diag(const GateLaunch& g, cudaStream_t s, int num_sms) {
  DiagParams<Real, KD> p;
  std::memset(&p, 0, sizeof p);
  p.re = static_cast<Real*>(g.re);
  p.im = static_cast<Real*>(g.im);
  p.n_work = (uint64_t{1} << (g.n - g.n_ctrl)) / V;
  p.fixed_or = g.fixed_or;
  p.n_ctrl = g.n_ctrl;
  for (int i = 0; i < g.n_ctrl; ++i) p.ctrl[i] = g.ctrl[i];
  for (int b = 0; b < KD; ++b) p.tq[b] = g.sub_targets[b];
  constexpr int D = 1 << KD;
  for (int j = 0; j < D; ++j) {
    p.dre[j] = static_cast<Real>(g.m_re[j * D + j]);
    p.dim[j] = static_cast<Real>(g.m_im[j * D + j]);
  }
  k_diag<Real, KD, V><<<grid_for(p.n_work, num_sms), 256, 0, s>>>(p);
  cuda_check(cudaGetLastError(), "k_diag launch");
}

template <typename Real>
void run_diag_wide(const GateLaunch& g, cudaStream_t s, int num_sms) {
  DiagWideParams<Real> p;
  std::memset(&p, 0, sizeof p);
  p.re = static_cast<Real*>(g.re);
  p.im = static_cast<Real*>(g.im);
  p.table = static_cast<const double*>(g.dev_mat);
  if (!p.table) throw std::runtime_error("wide diagonal launched without a device table");
  p.fixed_or = g.fixed_or;
  p.n_ctrl = g.n_ctrl;
  p.ks = g.ks;
  for (int i = 0; i < g.n_ctrl; ++i) p.ctrl[i] = g.ctrl[i];
  for (int b = 0; b < g.ks; ++b) p.tq[b] = g.sub_targets[b];
  p.full_range = g.full_range;
  if (g.full_range) {
    p.n_work = uint64_t{1} << (g.n - g.n_ctrl);
  } else {
    p.g_begin = g.g_begin;
    p.n_work = (g.g_end - g.g_begin) << g.ks;
    p.n_masks = g.n_masks;
    for (int i = 0; i < g.n_masks; ++i) p.masks[i] = g.masks[i];
  }
  if (p.n_work == 0) return;
  k_diag_wide<Real><<<grid_for(p.n_work, num_sms), 256, 0, s>>>(p);
  cuda_check(cudaGetLastError(), "k_diag_wide launch");
}

template <typename Real, int KD>
void pick_diag(const GateLaunch& g, cudaStream_t s, int num_sms) {
  const int low_ctrl = g.n_ctrl > 0 ? g.ctrl[0] : 64;
  const int active_bits = g.n - g.n_ctrl;
  if constexpr (PrecisionTraits<Real>::kMaxV >= 4) {
    if (low_ctrl >= 2 && active_bits >= 2) return run_diag<Real, KD, 4>(g, s, num_sms);
  }
  if (low_ctrl >= 1 && active_bits >= 1) return run_diag<Real, KD, 2>(g, s, num_sms);
  run_diag<Real, KD, 1>(g, s, num_sms);
}

// ------------------------------------------------------------------- tile
template <typename Real, int KS, int G, int RT, int GT>
void run_tile(const GateLaunch& g, cudaStream_t s, int num_sms) {
  using Shape = TileShape<Real, KS, G, RT, GT>;
  TileParams<Real> p;
  std::memset(&p, 0, sizeof p);
  p.re = static_cast<Real*>(g.re);
  p.im = static_cast<Real*>(g.im);
  p.mat = static_cast<const double*>(g.dev_mat);
  if (!p.mat) throw std::runtime_error("tile kernel launched without a device matrix");
  p.g_begin = g.g_begin;
  p.n_groups = g.g_end - g.g_begin;
  p.n_tiles = (p.n_groups + G - 1) / G;
  p.fixed_or = g.fixed_or;
  p.n_masks = g.n_masks;
  for (int i = 0; i < g.n_masks; ++i) p.masks[i] = g.masks[i];
  // dev_mat rows / columns are in the launch's element order (GateLaunch::perm,
  // chosen for the DMMA kernels; this kernel runs when their tile geometry
  // does not fit, e.g. states smaller than one DMMA tile)
  for (int j = 0; j < (1 << KS); ++j) p.off[j] = g.off[g.perm[j]];
  if (p.n_tiles == 0) return;
  auto kern = k_tile<Real, KS, G, RT, GT>;
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Shape::kSmem),
               "k_tile smem attribute");
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, Shape::kSmem), "k_tile occupancy");
    per_sm = std::max(per_sm, 1);
    configured = true;
  }
  const uint64_t blocks = std::min<uint64_t>(p.n_tiles, uint64_t(num_sms) * per_sm);
  kern<<<static_cast<unsigned>(blocks), 256, Shape::kSmem, s>>>(p);
  cuda_check(cudaGetLastError(), "k_tile launch");
}

template <typename Real>
void pick_tile(const GateLaunch& g, cudaStream_t s, int num_sms) {
  switch (g.ks) {
    case 5: return run_tile<Real, 5, 64, 2, 4>(g, s, num_sms);
    case 6:
      if constexpr (sizeof(Real) == 8) return run_tile<Real, 6, 32, 4, 2>(g, s, num_sms);
      else return run_tile<Real, 6, 64, 4, 4>(g, s, num_sms);
    default: throw std::runtime_error("tile kernel needs ks in {5, 6}");
  }
}

// ----------------------------------------------------------------- stream
// Tile geometry of k_stream for a full-range launch; false if the state is
// too small for one tile of the required shape.
template <typename Real, int KS>
bool stream_geometry(const GateLaunch& g, StreamParams<Real, KS>& p, size_t* smem, int* stages) {
  using S = StreamShape<KS>;
  int tg[24], nt = 0;  // all targets (controls + sub-targets), ascending
  {
    int a = 0, b = 0;
    while (a < g.n_ctrl || b < g.ks) {
      if (b >= g.ks || (a < g.n_ctrl && g.ctrl[a] < g.sub_targets[b])) tg[nt++] = g.ctrl[a++];
      else tg[nt++] = g.sub_targets[b++];
    }
  }
  int L = S::LOG2G;
  for (;;) {
    int below = 0;
    for (int i = 0; i < nt; ++i) below += tg[i] < L;
    if (S::LOG2G + below == L) break;
    L = S::LOG2G + below;
  }
  int n_low = 0, high_pos[24], n_high = 0, run_pos[8], n_run = 0;
  for (int i = 0; i < nt; ++i) {
    if (tg[i] < L) ++n_low;
    else high_pos[n_high++] = tg[i] - L;
  }
  for (int b = 0; b < g.ks; ++b)
    if (g.sub_targets[b] >= L) run_pos[n_run++] = g.sub_targets[b];
  if (L + n_high > g.n) return false;
  const int tile_bits = g.n - L - n_high;
  p.n_tiles = uint64_t{1} << tile_bits;
  p.L = L;
  p.n_runs = 1 << n_run;
  p.ctrl_or = g.fixed_or;
  p.n_tmask = insertion_masks(high_pos, n_high, tile_bits, p.tmask);
  int low_pos[24];
  for (int i = 0; i < n_low; ++i) low_pos[i] = tg[i];
  uint64_t gm[kMaxMasks + 12];
  p.n_gmask = insertion_masks(low_pos, n_low, S::LOG2G, gm);
  if (p.n_gmask > kMaxMasks || p.n_tmask > kMaxMasks) return false;
  for (int i = 0; i < p.n_gmask; ++i) p.gmask[i] = static_cast<uint32_t>(gm[i]);
  for (int r = 0; r < p.n_runs; ++r) {
    uint64_t o = 0;
    for (int b = 0; b < n_run; ++b) o |= static_cast<uint64_t>((r >> b) & 1) << run_pos[b];
    p.roff[r] = o;
  }
  for (int j = 0; j < (1 << KS); ++j) {
    uint32_t low = 0, run = 0;
    int hb = 0;
    for (int b = 0; b < KS; ++b) {
      const uint32_t bit = (j >> b) & 1u;
      if (g.sub_targets[b] < L) low |= bit << g.sub_targets[b];
      else run |= bit << hb++;
    }
    p.soff[j] = (run << L) + low;
  }
  const size_t stage = 2 * (size_t{1} << L) * p.n_runs * sizeof(Real);
  *stages = 3 * stage + 64 <= 200 * 1024 ? 3 : 2;
  *smem = *stages * stage + 64;
  return *smem <= 220 * 1024;
}

template <typename Real, int KS, int STAGES, bool SP>
void launch_stream(const StreamParams<Real, KS>& p, size_t smem, cudaStream_t s, int num_sms) {
  auto kern = k_stream<Real, KS, STAGES, SP>;
  static size_t configured_smem = 0;
  static int per_sm = 1;
  if (configured_smem < smem) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "k_stream smem");
    configured_smem = smem;
  }
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, StreamShape<KS>::kThreads, smem),
             "k_stream occupancy");
  const uint64_t blocks = std::min<uint64_t>(p.n_tiles, uint64_t(num_sms) * std::max(per_sm, 1));
  kern<<<static_cast<unsigned>(blocks), StreamShape<KS>::kThreads, smem, s>>>(p);
  cuda_check(cudaGetLastError(), "k_stream launch");
}

template <typename Real, int KS>
bool try_stream(const GateLaunch& g, cudaStream_t s, int num_sms) {
  StreamParams<Real, KS> p;
  std::memset(&p, 0, sizeof p);
  size_t smem = 0;
  int stages = 3;
  if (!stream_geometry<Real, KS>(g, p, &smem, &stages)) return false;
  p.re = static_cast<Real*>(g.re);
  p.im = static_cast<Real*>(g.im);
  constexpr int D = 1 << KS;
  for (int e = 0; e < D * D; ++e) {
    p.mr[e] = static_cast<Real>(g.m_re[e]);
    p.mi[e] = static_cast<Real>(g.m_im[e]);
    p.ms[e] = static_cast<Real>(g.m_re[e] + g.m_im[e]);
    if (p.mr[e] != Real(0)) p.nz[(3 * e) >> 5] |= 1u << ((3 * e) & 31);
    if (p.mi[e] != Real(0)) p.nz[(3 * e + 1) >> 5] |= 1u << ((3 * e + 1) & 31);
    if (p.ms[e] != Real(0)) p.nz[(3 * e + 2) >> 5] |= 1u << ((3 * e + 2) & 31);
  }
  if (stages == 3) {
    g.sparse ? launch_stream<Real, KS, 3, true>(p, smem, s, num_sms) : launch_stream<Real, KS, 3, false>(p, smem, s, num_sms);
  } else {
    g.sparse ? launch_stream<Real, KS, 2, true>(p, smem, s, num_sms) : launch_stream<Real, KS, 2, false>(p, smem, s, num_sms);
  }
  return true;
}

// ------------------------------------------------------------ stream_dmma
// TSG_DMMA_TMA: 0 off, 1 loads of the direct-out (FP64-bound) kernels,
// 2 loads of every kernel, 3 loads and write-backs
inline int dmma_tma_mode() {
  static const int mode = [] {
    const char* e = std::getenv("TSG_DMMA_TMA");
    return e && *e ? std::atoi(e) : 1;
  }();
  return mode;
}

template <typename Real, int KS, int LOG2G_ = DShape<Real, KS>::LOG2G>
bool dmma_geometry(const GateLaunch& g, DmmaParams<Real, KS>& p, size_t* smem, int* stages, bool simt,
                   bool few_tiles = false) {
  constexpr int kLog2G = LOG2G_;  // groups per tile of the caller's kernel (DShape's by default)
  int tg[24], nt = 0;  // all targets (controls + sub-targets), ascending
  {
    int a = 0, b = 0;
    while (a < g.n_ctrl || b < g.ks) {
      if (b >= g.ks || (a < g.n_ctrl && g.ctrl[a] < g.sub_targets[b])) tg[nt++] = g.ctrl[a++];
      else tg[nt++] = g.sub_targets[b++];
    }
  }
  int L = kLog2G;
  for (;;) {
    int below = 0;
    for (int i = 0; i < nt; ++i) below += tg[i] < L;
    if (kLog2G + below == L) break;
    L = kLog2G + below;
  }
  // element bit b of the launch's element order (GateLaunch::perm, a qubit
  // permutation) is qubit st[b]; runs follow the same order, so the smem
  // layout of the permuted gate is that of a gate on targets st[]
  int st[8];
  for (int b = 0; b < g.ks; ++b) st[b] = g.sub_targets[__builtin_ctz(static_cast<unsigned>(g.perm[1 << b]))];
  int n_low = 0, high_pos[24], n_high = 0, run_pos[8], n_run = 0, low_pos[24];
  for (int i = 0; i < nt; ++i) {
    if (tg[i] < L) low_pos[n_low++] = tg[i];
    else high_pos[n_high++] = tg[i] - L;
  }
  for (int b = 0; b < g.ks; ++b)
    if (st[b] >= L) run_pos[n_run++] = st[b];
  if (L + n_high > g.n) return false;
  const int tile_bits = g.n - L - n_high;
  p.n_tiles = uint64_t{1} << tile_bits;
  p.L = L;
  p.n_runs = 1 << n_run;
  const uint64_t low_mask = (uint64_t{1} << L) - 1;
  p.ctrl_hi = g.fixed_or & ~low_mask;
  p.ctrl_lo = static_cast<uint32_t>(g.fixed_or & low_mask);
  p.n_tmask = insertion_masks(high_pos, n_high, tile_bits, p.tmask);
  uint64_t gm[kMaxMasks + 12];
  p.n_gmask = insertion_masks(low_pos, n_low, kLog2G, gm);
  if (p.n_gmask > kMaxMasks || p.n_tmask > kMaxMasks) return false;
  for (int i = 0; i < p.n_gmask; ++i) p.gmask[i] = static_cast<uint32_t>(gm[i]);
  for (int r = 0; r < p.n_runs; ++r) {
    uint64_t o = 0;
    for (int b = 0; b < n_run; ++b) o |= static_cast<uint64_t>((r >> b) & 1) << run_pos[b];
    p.roff[r] = o;
  }
  uint32_t low_of[1 << KS], run_of[1 << KS];
  for (int j = 0; j < (1 << KS); ++j) {
    uint32_t low = 0, run = 0;
    int hb = 0;
    for (int b = 0; b < KS; ++b) {
      const uint32_t bit = (j >> b) & 1u;
      if (st[b] < L) low |= bit << st[b];
      else run |= bit << hb++;
    }
    low_of[j] = low;
    run_of[j] = run;
    p.goff[j] = p.roff[run] + low;
  }
  // Shared-memory layout: runs padded by kRunPadBytes; a long run whose B
  // fragments (8 groups x 4 elements per warp load) would pile onto few
  // banks is cut into padded 256-byte chunks instead (e.g. targets 0..4: all
  // groups 256 bytes apart).  Pick the layout with fewer wavefronts.
  const uint32_t pad = kRunPadBytes / sizeof(Real);
  auto layout = [&](int chunk_log2, uint32_t* chunk_stride, uint32_t* run_stride) {
    *chunk_stride = (1u << chunk_log2) + pad;
    *run_stride = chunk_log2 == L ? *chunk_stride : (1u << (L - chunk_log2)) * *chunk_stride;
  };
  auto wavefronts = [&](int chunk_log2) {  // B-fragment load of warp 0, k-step 0
    uint32_t cs, rs;
    layout(chunk_log2, &cs, &rs);
    auto padw = [&](uint32_t w) { return (w >> chunk_log2) * cs + (w & ((1u << chunk_log2) - 1)); };
    int worst = 0;
    for (int k = 0; k < (1 << KS) / 4; ++k) {
      int words[32] = {0};
      for (int lane = 0; lane < 32; ++lane) {
        const int lr = lane >> 2, lc = lane & 3;
        uint32_t gpos = 0;
        for (int i = 0; i < p.n_gmask; ++i) gpos += (static_cast<uint32_t>(lr) & p.gmask[i]) << i;
        gpos |= p.ctrl_lo;
        const int j = 4 * k + lc;
        const uint32_t a = run_of[j] * rs + padw(low_of[j]) + padw(gpos);  // element offset (Real units)
        const uint32_t w = a * (sizeof(Real) / 4);
        for (uint32_t b = 0; b < sizeof(Real) / 4; ++b) ++words[(w + b) % 32];
      }
      for (int b = 0; b < 32; ++b) worst = std::max(worst, words[b]);
    }
    return worst;
  };
  p.chunk_log2 = L;
  // 256-byte chunks; complex128 products with at most half of their 8 x 4
  // tiles nonzero are bound by the producer's copy issue rather than by the
  // B-fragment loads: 512-byte chunks (half the bulk copies; RQC-30's
  // 5-qubit launches 186 -> 179 ms, dense ones measured better at 256)
  const int chunk = sizeof(Real) == 8 ? (few_tiles ? 6 : 5) : 6;
  // only for ks = 5, whose stages are loaded and never bulk-stored: more,
  // smaller bulk copies measured slower for the HBM-bound ks <= 4 kernels
  const bool direct_out = KS >= 5 || (sizeof(Real) == 4 && KS >= 4);  // k_stream_dmma kDirectOut
  if (direct_out && !simt && L > chunk && wavefronts(chunk) < wavefronts(L)) p.chunk_log2 = chunk;
  // TMA tile loads (dmma_tma_plan) take boxes of at most 256 elements per
  // row: a longer padded run is cut into the chunk size with the fewest
  // wavefronts instead
  if (direct_out && !simt && dmma_tma_mode() >= 1 && p.chunk_log2 == L && (1u << L) + pad > 256 && n_run > 0) {
    int best = 7;
    for (int c = 6; c >= 5; --c)
      if (wavefronts(c) < wavefronts(best)) best = c;
    p.chunk_log2 = best;
  }
  layout(p.chunk_log2, &p.chunk_stride, &p.run_stride);
  for (int j = 0; j < (1 << KS); ++j) {
    const uint32_t w = low_of[j];
    p.soff[j] = run_of[j] * p.run_stride + (w >> p.chunk_log2) * p.chunk_stride + (w & ((1u << p.chunk_log2) - 1));
  }
  // one run, one chunk: the padding after it serves no bank spread, and
  // without it the run is a plain (TMA-expressible) box
  if (p.n_runs == 1 && p.chunk_log2 == L) p.chunk_stride = p.run_stride = 1u << L;
  // stages start on 128-byte boundaries (TMA tensor-copy destinations)
  constexpr uint32_t kAlignElems = 128 / sizeof(Real);
  p.stage_elems = (p.run_stride * static_cast<uint32_t>(p.n_runs) + kAlignElems - 1) / kAlignElems * kAlignElems;
  // Two CTAs per SM beat deeper pipelines (measured): 3 stages when two CTAs
  // still fit in shared memory, else 2.
  const size_t stage = 2 * size_t{p.stage_elems} * sizeof(Real);
  size_t fixed = 128;  // (complex64 6-qubit geometries serve k_stream_umma, which sizes its own shared memory)
  if constexpr (KS <= 5) fixed += simt ? dmma_m_smem_bytes<Real, KS, true>() : dmma_m_smem_bytes<Real, KS>();
  if constexpr (KS == 6 && sizeof(Real) == 8) fixed += dmma_m_smem_bytes<Real, KS>();
  const size_t per_cta = 110 * 1024;
  *stages = 3 * stage + fixed <= per_cta ? 3 : 2;
  *smem = *stages * stage + fixed;
  return *smem <= 220 * 1024;
}

// TMA tensor maps for a k_stream_dmma launch (DmmaParams::tmap): the tile's
// shared-memory layout [runs][chunks][chunk + pad] is one box of a rank-5
// view of the state --
//   dim 0  the chunk's amplitudes; the box is pad elements wider than the
//          dimension, so the padding is zero-filled on loads and skipped on
//          stores (an unchunked, unpadded run: up to 256 amplitudes, dim 1
//          takes the rest)
//   dim 1  chunks of a run
//   dim 2  tile base >> L (box 1): the tile bases and the run offsets are
//          disjoint index bits, so this dimension aliases the next two
//   dim 3, 4  the lowest run bits, as runs of consecutive qubits
// -- and runs beyond dims 3-4 take one copy each (tma_issues).  Needs 128-byte
// aligned copy destinations and box widths of at most 256 elements; returns
// false (per-chunk bulk copies) otherwise.  TSG_DMMA_TMA=0 disables.
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

template <typename Real, int KS>
bool dmma_tma_plan(const GateLaunch& g, DmmaParams<Real, KS>& p) {
  static_assert(sizeof(TmaDesc) == sizeof(CUtensorMap), "TmaDesc mirrors CUtensorMap");
  p.tma_issues = p.tma_store = 0;
  const int mode = dmma_tma_mode();
  const bool direct_out = KS >= 5 || (sizeof(Real) == 4 && KS >= 4);  // k_stream_dmma kDirectOut
  if (mode <= 0 || (mode == 1 && !direct_out) || !tensor_map_encoder()) return false;
  const uint32_t e0 = 1u << p.chunk_log2, pad = p.chunk_stride - e0;
  cuuint64_t dim[5] = {1, 1, 1, 1, 1}, stride[4] = {0, 0, 0, 0};
  cuuint32_t box[5] = {1, 1, 1, 1, 1}, estride[5] = {1, 1, 1, 1, 1};
  if (pad == 0) {  // one unpadded run: contiguous 2^L amplitudes
    const uint32_t d0 = std::min<uint32_t>(1u << p.L, 256);
    dim[0] = box[0] = d0;
    dim[1] = box[1] = (1u << p.L) / d0;
    stride[0] = size_t{d0} * sizeof(Real);
  } else {
    if (e0 + pad > 256) return false;
    dim[0] = e0;
    box[0] = e0 + pad;
    dim[1] = box[1] = 1u << (p.L - p.chunk_log2);
    stride[0] = size_t{e0} * sizeof(Real);
  }
  if (size_t{box[0]} * sizeof(Real) % 16 != 0) return false;
  dim[2] = uint64_t{1} << (g.n - p.L);
  stride[1] = (size_t{1} << p.L) * sizeof(Real);
  // run bit b is qubit ctz(roff[1 << b]); dims 3 and 4 take the lowest two
  // groups of consecutive qubits
  int n_run = 0;
  while ((1 << n_run) < p.n_runs) ++n_run;
  int b = 0;
  for (int d = 3; d <= 4 && b < n_run; ++d) {
    const int q0 = __builtin_ctzll(p.roff[1 << b]);
    int m = 1;
    while (b + m < n_run && __builtin_ctzll(p.roff[1 << (b + m)]) == q0 + m) ++m;
    dim[d] = box[d] = 1u << m;
    stride[d - 1] = (size_t{1} << q0) * sizeof(Real);
    b += m;
  }
  for (int d = 2; d < 4; ++d)
    if (stride[d] == 0) stride[d] = stride[d - 1];  // unused (size 1) dimensions
  p.tma_shift = b;
  p.tma_issue_elems = (1u << b) * p.run_stride;
  const int issues = p.n_runs >> b;
  if (issues > 1 && (p.tma_issue_elems * sizeof(Real)) % 128 != 0) return false;
  if ((reinterpret_cast<uintptr_t>(g.re) | reinterpret_cast<uintptr_t>(g.im)) & 15u) return false;
  const CUtensorMapDataType type = sizeof(Real) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  for (int a = 0; a < 2; ++a) {
    void* base = a ? g.im : g.re;
    if (tensor_map_encoder()(reinterpret_cast<CUtensorMap*>(&p.tmap[a]), type, 5, base, dim, stride, box, estride,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  p.tma_issues = issues;
  p.tma_store = mode >= 3 && !direct_out;
  return true;
}

template <typename Real, int KS, int STAGES, bool SP, bool SIMT, bool TPOSE = false>
void launch_dmma(const DmmaParams<Real, KS>& p, size_t smem, cudaStream_t s, int num_sms) {
  auto kern = k_stream_dmma<Real, KS, STAGES, SP, SIMT, TPOSE>;
  static size_t configured_smem = 0;
  if (configured_smem < smem) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "dmma smem");
    configured_smem = smem;
  }
  int per_sm = 1;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, DShape<Real, KS>::kThreads + 32, smem),
             "dmma occupancy");
  const uint64_t blocks = std::min<uint64_t>(p.n_tiles, uint64_t(num_sms) * std::max(per_sm, 1));
  kern<<<static_cast<unsigned>(blocks), DShape<Real, KS>::kThreads + 32, smem, s>>>(p);
  cuda_check(cudaGetLastError(), "k_stream_dmma launch");
}

template <typename Real, int KS, int STAGES, bool SP>
void launch_dmma_pick(const DmmaParams<Real, KS>& p, size_t smem, cudaStream_t s, int num_sms, bool simt, bool tpose) {
  if constexpr (sizeof(Real) == 4 && KS <= 3) {
    if (simt) return launch_dmma<Real, KS, STAGES, false, true>(p, smem, s, num_sms);  // SIMT evaluates densely
  }
  if constexpr (KS == 5 || (sizeof(Real) == 4 && KS == 4)) {
    if (tpose) return launch_dmma<Real, KS, STAGES, SP, false, true>(p, smem, s, num_sms);
  }
  if constexpr (KS >= 6) launch_dmma<Real, KS, STAGES, false, false>(p, smem, s, num_sms);
  else launch_dmma<Real, KS, STAGES, SP, false>(p, smem, s, num_sms);
}

// Host half of a k_stream_dmma launch: nonzero tile masks, variant,
// geometry (no device pointers needed).
template <typename Real, int KS>
struct DmmaSetup {
  DmmaParams<Real, KS> p;
  size_t smem = 0;
  int stages = 3;
  bool simt = false, sparse = false;
  bool tpose = false;  // transposed product (k_stream_dmma TPOSE): qubit 0 is the first element bit
  int nonzero = 0;     // nonzero 8 x 4 tiles of [Mr | Mi | Ms]
};

template <typename Real, int KS>
bool dmma_setup(const GateLaunch& g, DmmaSetup<Real, KS>& st) {
  using S = DShape<Real, KS>;
  DmmaParams<Real, KS>& p = st.p;
  std::memset(&p, 0, sizeof p);
  // complex64, 3 qubits, every target and control at bit 5 or above: FP32
  // SIMT consumer (measured faster there; slower than the FP64-widened DMMA
  // product for 4-5 qubits and for low targets -- scripts/pass_bench.py)
  int lowest = 64;
  for (int b = 0; b < g.ks; ++b) lowest = std::min(lowest, g.sub_targets[b]);
  for (int c = 0; c < g.n_ctrl; ++c) lowest = std::min(lowest, g.ctrl[c]);
  st.simt = sizeof(Real) == 4 && KS <= 3 && lowest >= 5;
  // direct-out products whose first element bit is qubit 0: two groups are
  // never adjacent there, two elements are -- the transposed product stores
  // 2-element vectors (TSG_DMMA_TPOSE=0 disables)
  static const bool tpose_on = [] {
    const char* e = std::getenv("TSG_DMMA_TPOSE");
    return !(e && e[0] == '0');
  }();
  const bool direct_out = KS >= 5 || (sizeof(Real) == 4 && KS >= 4);  // k_stream_dmma kDirectOut
  st.tpose = tpose_on && direct_out && KS <= 5 && !st.simt && g.sub_targets[__builtin_ctz(static_cast<unsigned>(g.perm[1]))] == 0;
  constexpr int D = S::D;
  for (int rb = 0; rb < S::RB; ++rb)
    for (int k = 0; k < S::KST && KS <= 5; ++k) {  // (ks = 6: dense only)
      bool nzr = false, nzi = false, nzs = false;
      for (int r = 8 * rb; r < 8 * rb + 8; ++r)
        for (int c = 4 * k; c < 4 * k + 4; ++c) {
          const int e = g.perm[r] * D + g.perm[c];
          nzr |= g.m_re[e] != 0.0;
          nzi |= g.m_im[e] != 0.0;
          nzs |= (g.m_re[e] + g.m_im[e]) != 0.0;
        }
      const int bit = rb * S::KST + k;
      p.nzblk[0] |= static_cast<uint32_t>(nzr) << bit;
      p.nzblk[1] |= static_cast<uint32_t>(nzi) << bit;
      p.nzblk[2] |= static_cast<uint32_t>(nzs) << bit;
    }
  // The sparse variant (per-tile predicates) pays only when it skips at least
  // a quarter of the DMMAs: RQC-30's 5-qubit gates with 28/32 nonzero tiles ran
  // 8-10 ms sparse, 7.7-8.4 ms dense (scripts/ks5_rqc_sparse.py); skipped zero
  // tiles would only have added exact zeros.  (A JIT kernel with the masks
  // compiled in skips every zero tile at no cost: dmma_jit_spec.)
  const int n_dmma_tiles = 3 * S::RB * S::KST;
  st.nonzero = KS <= 5 ? __builtin_popcount(p.nzblk[0]) + __builtin_popcount(p.nzblk[1]) + __builtin_popcount(p.nzblk[2])
                       : n_dmma_tiles;
  static const bool any_zero_rule = std::getenv("TSG_DMMA_SPARSE_ANY") != nullptr;  // round-1 rule (A/B runs)
  st.sparse = KS <= 5 && (any_zero_rule ? st.nonzero < n_dmma_tiles : 4 * (n_dmma_tiles - st.nonzero) >= n_dmma_tiles);
  static const int force_sparse = [] {  // experiments: TSG_DMMA_SPARSE=0|1 forces the variant
    const char* e = std::getenv("TSG_DMMA_SPARSE");
    return e ? std::atoi(e) : -1;
  }();
  if (force_sparse >= 0 && KS <= 5) st.sparse = force_sparse == 1;
  const int most = std::max({__builtin_popcount(p.nzblk[0]), __builtin_popcount(p.nzblk[1]), __builtin_popcount(p.nzblk[2])});
  return dmma_geometry<Real, KS>(g, p, &st.smem, &st.stages, st.simt, KS <= 5 && 2 * most <= S::RB * S::KST);
}

// a JIT-compiled product (dmma_jit_spec): same parameters and geometry
template <typename Real, int KS>
void launch_dmma_jit(const void* kern, const DmmaParams<Real, KS>& p, size_t smem, cudaStream_t s, int num_sms) {
  using S = DShape<Real, KS>;
  cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
             "dmma jit smem");
  int per_sm = 1;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::kThreads + 32, smem), "dmma jit occupancy");
  const uint64_t blocks = std::min<uint64_t>(p.n_tiles, uint64_t(num_sms) * std::max(per_sm, 1));
  DmmaParams<Real, KS> arg = p;
  void* args[] = {&arg};
  cuda_check(cudaLaunchKernel(kern, dim3(static_cast<unsigned>(blocks)), dim3(S::kThreads + 32), args, smem, s),
             "k_stream_dmma jit launch");
}

template <typename Real, int KS>
bool try_dmma(const GateLaunch& g, cudaStream_t s, int num_sms) {
  using S = DShape<Real, KS>;
  if (!g.dev_mat) return false;
  DmmaSetup<Real, KS> st;
  if (!dmma_setup<Real, KS>(g, st)) return false;
  DmmaParams<Real, KS>& p = st.p;
  p.re = static_cast<Real*>(g.re);
  p.im = static_cast<Real*>(g.im);
  p.mat = static_cast<const double*>(g.dev_mat);
  dmma_tma_plan<Real, KS>(g, p);
  static const bool debug = std::getenv("TSG_DMMA_DEBUG") != nullptr;
  if (debug)
    std::fprintf(stderr, "dmma ks=%d L=%d chunk=%d runs=%d tma=%d tpose=%d stages=%d smem=%zu tiles=%d/%d/%d of %d sparse=%d jit=%d\n",
                 KS, p.L, p.chunk_log2, p.n_runs, p.tma_issues, st.tpose ? 1 : 0, st.stages, st.smem, __builtin_popcount(p.nzblk[0]),
                 __builtin_popcount(p.nzblk[1]), __builtin_popcount(p.nzblk[2]), S::RB * S::KST, st.sparse ? 1 : 0,
                 g.jit ? 1 : 0);
  if constexpr (sizeof(Real) == 8 && KS <= 5) {
    if (g.jit) {
      launch_dmma_jit<Real, KS>(g.jit, p, st.smem, s, num_sms);
      return true;
    }
  }
  switch (st.stages) {
    case 3:
      st.sparse ? launch_dmma_pick<Real, KS, 3, true>(p, st.smem, s, num_sms, st.simt, st.tpose)
                : launch_dmma_pick<Real, KS, 3, false>(p, st.smem, s, num_sms, st.simt, st.tpose);
      break;
    default:
      st.sparse ? launch_dmma_pick<Real, KS, 2, true>(p, st.smem, s, num_sms, st.simt, st.tpose)
                : launch_dmma_pick<Real, KS, 2, false>(p, st.smem, s, num_sms, st.simt, st.tpose);
      break;
  }
  return true;
}

// ---------------------------------------------------------- stream_umma
// complex64 4- and 5-qubit sub-gates on the INT8 tensor cores
// (kernels_umma.cuh).  TSG_UMMA=0 disables it (the FP64-widened DMMA product
// runs instead); TSG_UMMA_KS=<bitmask of ks> overrides which sizes take it.
inline uint32_t umma_ks_mask() {
  static uint32_t mask = [] {
    const char* e = std::getenv("TSG_UMMA");
    if (e && std::string(e) == "0") return 0u;
    const char* m = std::getenv("TSG_UMMA_KS");
    return (m ? static_cast<uint32_t>(std::strtoul(m, nullptr, 0)) : TSG_UMMA_DEFAULT_KS) & 0x70u;
  }();
  return mask;
}

template <int KS, int STAGES>
void launch_umma(const DmmaParams<float, KS>& p, size_t smem, cudaStream_t s, int num_sms) {
  using U = UmmaShape<KS>;
  auto kern = k_stream_umma<KS, STAGES>;
  static size_t configured_smem = 0;
  if (configured_smem < smem) {
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "umma smem");
    configured_smem = smem;
  }
  const uint64_t blocks = std::min<uint64_t>(p.n_tiles, uint64_t(num_sms) * U::kCtasPerSm);
  kern<<<static_cast<unsigned>(blocks), U::T + 32, smem, s>>>(p);
  cuda_check(cudaGetLastError(), "k_stream_umma launch");
}

// Geometry of a k_stream_umma launch, or false when the gate stays on the
// DMMA product.  Lanes own consecutive groups, so low targets / controls
// spread a warp's stage reads over few banks and its global stores over more
// sectors: with a target or control on bit 0 the tensor-core kernel only
// takes gates whose lanes stay (nearly) contiguous, e.g. [0, 7, 14, 21, 28]
// (4.0 ms vs 8.1 ms for the DMMA product; [0, 1, 2, 3]: 11.4 vs 7.4 ms).
template <int KS>
bool umma_plan(const GateLaunch& g, DmmaParams<float, KS>& p) {
  if (!g.dev_mat || !g.full_range || !((umma_ks_mask() >> KS) & 1u)) return false;
  std::memset(&p, 0, sizeof p);
  size_t dsmem = 0;
  int dstages = 0;
  // geometry without chunked runs (the simt layout): one bulk copy per run
  if (!dmma_geometry<float, KS, UmmaShape<KS>::LOG2G>(g, p, &dsmem, &dstages, /*simt=*/true)) return false;
  if (p.chunk_log2 != p.L) return false;
  // most words any bank receives from the 32 lanes' first stage read
  auto degree = [&](int chunk_log2, uint32_t chunk_stride) {
    int words[32] = {0}, worst = 0;
    for (uint32_t l = 0; l < 32; ++l) {
      uint32_t gp = 0;
      for (int i = 0; i < p.n_gmask; ++i) gp += (l & p.gmask[i]) << i;
      gp |= p.ctrl_lo;
      const uint32_t a = (gp >> chunk_log2) * chunk_stride + (gp & ((1u << chunk_log2) - 1));
      worst = std::max(worst, ++words[a % 32]);
    }
    return worst;
  };
  const int d0 = degree(p.L, p.run_stride);
  bool bit0 = false;
  for (int b = 0; b < g.ks; ++b) bit0 |= g.sub_targets[b] == 0;
  for (int c = 0; c < g.n_ctrl; ++c) bit0 |= g.ctrl[c] == 0;
  // (6 qubits have no DMMA product to fall back to: k_tile is ~3x slower
  // than even a bank-conflicted tensor-core launch)
  if (bit0 && d0 > 2 && KS <= 5) return false;
  // Runs whose stage reads would pile 16 or more lanes onto one bank are cut
  // into padded 64-amplitude chunks (more, smaller bulk copies: measured
  // slower below that conflict degree)
  static const bool chunking = !std::getenv("TSG_UMMA_NO_CHUNK");
  const uint32_t cstride = 64 + kRunPadBytes / sizeof(float);
  const int d6 = p.L > 6 ? degree(6, cstride) : d0;
  if (chunking && p.L > 6 && d0 >= 16 && (d6 <= 4 || (KS == 6 && 2 * d6 <= d0))) {
    uint32_t low_of[1 << KS], run_of[1 << KS];
    for (int j = 0; j < (1 << KS); ++j) {  // each element's run and in-run offset
      run_of[j] = p.soff[j] / p.run_stride;
      low_of[j] = p.soff[j] % p.run_stride;
    }
    p.chunk_log2 = 6;
    p.chunk_stride = cstride;
    p.run_stride = (1u << (p.L - 6)) * p.chunk_stride;
    for (int j = 0; j < (1 << KS); ++j)
      p.soff[j] = run_of[j] * p.run_stride + (low_of[j] >> 6) * p.chunk_stride + (low_of[j] & 63u);
  }
  p.stage_elems = (p.run_stride * static_cast<uint32_t>(p.n_runs) + 31u) / 32u * 32u;  // 128-byte stages
  return true;
}

inline bool umma_takes(const GateLaunch& g) {
  if (g.ks == 4) {
    DmmaParams<float, 4> p;
    return umma_plan<4>(g, p);
  }
  if (g.ks == 5) {
    DmmaParams<float, 5> p;
    return umma_plan<5>(g, p);
  }
  if (g.ks == 6) {
    DmmaParams<float, 6> p;
    return umma_plan<6>(g, p);
  }
  return false;
}

template <int KS>
bool try_umma(const GateLaunch& g, cudaStream_t s, int num_sms) {
  DmmaParams<float, KS> p;
  if (!umma_plan<KS>(g, p)) return false;
  p.re = static_cast<float*>(g.re);
  p.im = static_cast<float*>(g.im);
  p.mat = static_cast<const double*>(g.dev_mat);
  dmma_tma_plan<float, KS>(g, p);
  // two CTAs per SM (256 TMEM columns each), two stages each; at least 80 KB
  // so that a third CTA never lands on an SM (tcgen05.alloc would wait)
  const size_t stage = 2 * size_t{p.stage_elems} * sizeof(float);
  const size_t fixed = umma_fixed_smem<KS>() + 256;
  if constexpr (UmmaShape<KS>::kCtasPerSm == 1) {  // one CTA per SM (all of TMEM): > 114 KB keeps it so
    if (fixed + 2 * stage > 227 * 1024) return false;
    launch_umma<KS, 2>(p, std::max(fixed + 2 * stage, size_t{120} * 1024), s, num_sms);
    return true;
  }
  static const int max_stages = std::getenv("TSG_UMMA_STAGES") ? std::atoi(std::getenv("TSG_UMMA_STAGES")) : 3;
  if (max_stages >= 3 && fixed + 3 * stage <= 113 * 1024) {
    launch_umma<KS, 3>(p, std::max(fixed + 3 * stage, size_t{80} * 1024), s, num_sms);
    return true;
  }
  if (fixed + 2 * stage > 113 * 1024) return false;
  launch_umma<KS, 2>(p, std::max(fixed + 2 * stage, size_t{80} * 1024), s, num_sms);
  return true;
}

// ---------------------------------------------------------- dmma_direct
template <int KS>
bool try_dmma_direct(const GateLaunch& g, cudaStream_t s, int num_sms) {
  using S = DdShape<KS>;
  if (!g.dev_mat) return false;
  const uint64_t count = g.g_end - g.g_begin;
  if (count % S::GI != 0 || count == 0) return false;
  DdParams<KS> p;
  std::memset(&p, 0, sizeof p);
  p.re = static_cast<double*>(g.re);
  p.im = static_cast<double*>(g.im);
  p.mat = static_cast<const double*>(g.dev_mat);
  p.g_begin = g.g_begin;
  p.n_items = count / S::GI;
  p.fixed_or = g.fixed_or;
  p.n_masks = g.n_masks;
  for (int i = 0; i < g.n_masks; ++i) p.masks[i] = g.masks[i];
  for (int j = 0; j < S::D; ++j) p.off[j] = g.off[g.perm[j]];  // element order of dev_mat
  bool all = true;
  for (int rb = 0; rb < S::RB; ++rb)
    for (int k = 0; k < S::KST; ++k) {
      bool nz[3] = {false, false, false};
      for (int r = 8 * rb; r < 8 * rb + 8; ++r)
        for (int c = 4 * k; c < 4 * k + 4; ++c) {
          const int e = g.perm[r] * S::D + g.perm[c];
          nz[0] |= g.m_re[e] != 0.0;
          nz[1] |= g.m_im[e] != 0.0;
          nz[2] |= (g.m_re[e] + g.m_im[e]) != 0.0;
        }
      for (int m = 0; m < 3; ++m) {
        p.nzblk[m] |= static_cast<uint32_t>(nz[m]) << (rb * S::KST + k);
        all &= nz[m];
      }
    }
  auto kern = all ? k_dmma_direct<KS, false> : k_dmma_direct<KS, true>;
  int per_sm = 1;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * S::kWarps, 0), "dmma_direct occupancy");
  const uint64_t blocks =
      std::min<uint64_t>((p.n_items + S::kWarps - 1) / S::kWarps, uint64_t(num_sms) * std::max(per_sm, 1));
  kern<<<static_cast<unsigned>(blocks), 32 * S::kWarps, 0, s>>>(p);
  cuda_check(cudaGetLastError(), "k_dmma_direct launch");
  return true;
}

inline int dmma_mode() {
  static int mode = [] {
    const char* e = std::getenv("TSG_DMMA_MODE");
    if (!e) return 0;
    return std::string(e) == "direct" ? 1 : (std::string(e) == "stream" ? 2 : 0);
  }();
  return mode;
}

// Full-range non-diagonal sub-gates of 3..5 qubits: complex128 on the DMMA
// pipe (k_stream_dmma or k_dmma_direct), complex64 ks=3 on the SIMT k_stream.
template <typename Real>
bool launch_stream_if(const GateLaunch& g, cudaStream_t s, int num_sms) {
  if (!g.full_range || (g.klass != 2 && g.klass != 3)) return false;
  if constexpr (sizeof(Real) == 8) {
    const bool direct = dmma_mode() == 1;
    switch (g.ks) {
      case 3: return direct ? try_dmma_direct<3>(g, s, num_sms) : try_dmma<double, 3>(g, s, num_sms);
      case 4: return direct ? try_dmma_direct<4>(g, s, num_sms) : try_dmma<double, 4>(g, s, num_sms);
      case 5: return direct ? try_dmma_direct<5>(g, s, num_sms) : try_dmma<double, 5>(g, s, num_sms);
      case 6: return try_dmma<double, 6>(g, s, num_sms);
      default: return false;
    }
  } else {
    switch (g.ks) {  // complex64: INT8 slices on tcgen05 (ks 4, 5), else widened to FP64 on the DMMA pipe
      case 3: return try_dmma<float, 3>(g, s, num_sms);
      case 4: return try_umma<4>(g, s, num_sms) || try_dmma<float, 4>(g, s, num_sms);
      case 5: return try_umma<5>(g, s, num_sms) || try_dmma<float, 5>(g, s, num_sms);
      case 6: return try_umma<6>(g, s, num_sms);
      default: return false;
    }
  }
}

// ---------------------------------------------------------- diag batches
template <typename Real>
int launch_diag_batch_impl(const DiagBatchLaunch& b, cudaStream_t s, int num_sms) {
  if (b.n_gates == 0) return 0;
  constexpr int V = PrecisionTraits<Real>::kMaxV;  // 16-byte vectors
  const uint64_t n_work = (uint64_t{1} << b.n) / V;
  if (n_work == 0 || (uint64_t{1} << b.n) % V != 0) throw std::runtime_error("diagonal batch needs >= 4 amplitudes");
  if (b.n <= 32) k_diag_batch<Real, V, uint32_t><<<grid_for(n_work, num_sms), 256, 0, s>>>(b, n_work);
  else k_diag_batch<Real, V, uint64_t><<<grid_for(n_work, num_sms), 256, 0, s>>>(b, n_work);
  cuda_check(cudaGetLastError(), "k_diag_batch launch");
  return 1;
}

// ------------------------------------------------------------------ entry
template <typename Real>
int launch_gate_impl(const GateLaunch& g, cudaStream_t s, int num_sms) {
  constexpr int DM = PrecisionTraits<Real>::kDirectMax;
  int klass = g.klass;
  if (klass == 0) return 0;
  if (klass == 1 && g.ks > kMaxSub) {
    run_diag_wide<Real>(g, s, num_sms);
    return 1;
  }
  if (launch_stream_if<Real>(g, s, num_sms)) return 1;
  if (klass == 1 && !g.full_range) klass = g.ks <= DM ? 2 : 3;  // sub-range: group-space kernels
  if (klass == 2 && g.ks > DM) klass = 3;
  if (klass == 1) {
    switch (g.ks) {
      case 0: pick_diag<Real, 0>(g, s, num_sms); break;
      case 1: pick_diag<Real, 1>(g, s, num_sms); break;
      case 2: pick_diag<Real, 2>(g, s, num_sms); break;
      case 3: pick_diag<Real, 3>(g, s, num_sms); break;
      case 4: pick_diag<Real, 4>(g, s, num_sms); break;
      case 5: pick_diag<Real, 5>(g, s, num_sms); break;
      case 6: pick_diag<Real, 6>(g, s, num_sms); break;
      default: throw std::runtime_error("diagonal sub-gate wider than 6 qubits");
    }
    return 1;
  }
  if (klass == 2) {
    switch (g.ks) {
      case 0: pick_direct<Real, 0>(g, s, num_sms); break;
      case 1: pick_direct<Real, 1>(g, s, num_sms); break;
      case 2: pick_direct<Real, 2>(g, s, num_sms); break;
      case 3: pick_direct<Real, 3>(g, s, num_sms); break;
      case 4: pick_direct<Real, 4>(g, s, num_sms); break;
      case 5:
        if constexpr (DM >= 5) {
          pick_direct<Real, 5>(g, s, num_sms);
          break;
        }
        [[fallthrough]];
      default: throw std::runtime_error("direct kernel sub-gate too wide");
    }
    return 1;
  }
  pick_tile<Real>(g, s, num_sms);
  return 1;
}

// Name of the kernel template launch_gate_impl selects for a full-range
// launch (reports / profiles), e.g. "k_stream_dmma<ks=5>".
// Whether k_stream_dmma's tile geometry fits the state (else launch_gate_impl
// falls through to k_tile / k_direct)
template <typename Real>
bool dmma_fits(const GateLaunch& g) {
  size_t smem = 0;
  int stages = 0;
  switch (g.ks) {
    case 3: {
      DmmaParams<Real, 3> p{};
      return dmma_geometry<Real, 3>(g, p, &smem, &stages, false);
    }
    case 4: {
      DmmaParams<Real, 4> p{};
      return dmma_geometry<Real, 4>(g, p, &smem, &stages, false);
    }
    case 5: {
      DmmaParams<Real, 5> p{};
      return dmma_geometry<Real, 5>(g, p, &smem, &stages, false);
    }
    case 6: {
      if constexpr (sizeof(Real) != 8) return false;
      DmmaParams<Real, 6> p{};
      return dmma_geometry<Real, 6>(g, p, &smem, &stages, false);
    }
    default:
      return false;
  }
}

template <typename Real>
std::string kernel_name_impl(const GateLaunch& g) {
  constexpr int DM = PrecisionTraits<Real>::kDirectMax;
  const std::string ks = "<ks=" + std::to_string(g.ks);
  int klass = g.klass;
  if (klass == 0) return "none";
  if (klass == 1 && g.ks > kMaxSub) return "k_diag_wide" + ks + ">";
  if ((klass == 2 || klass == 3) && sizeof(Real) == 4 && umma_takes(g)) return "k_stream_umma" + ks + ">";
  if (g.full_range && (klass == 2 || klass == 3) && g.ks >= 3 && (g.ks <= 5 || (g.ks == 6 && sizeof(Real) == 8)) &&
      g.dev_mat) {
    if (dmma_mode() == 1 && sizeof(Real) == 8 && g.ks <= 5) return "k_dmma_direct" + ks + ">";
    if (dmma_fits<Real>(g)) return "k_stream_dmma" + ks + ">";
  }
  if (klass == 1 && !g.full_range) klass = g.ks <= DM ? 2 : 3;
  if (klass == 2 && g.ks > DM) klass = 3;
  switch (klass) {
    case 1: return "k_diag" + ks + ">";
    case 2: return "k_direct" + ks + (g.sparse ? ",sparse>" : ",dense>");
    default: return "k_tile" + ks + ">";
  }
}

}  // namespace tsg
