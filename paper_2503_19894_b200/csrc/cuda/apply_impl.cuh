// Launch-side dispatch for one precision: GateLaunch -> kernel template
// instance + grid.  Included once per precision (apply_f64.cu, apply_f32.cu)
// so the two halves of the instantiation set compile in parallel.
#pragma once

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

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
  p.mat = static_cast<const Real*>(g.dev_mat);
  if (!p.mat) throw std::runtime_error("tile kernel launched without a device matrix");
  p.g_begin = g.g_begin;
  p.n_groups = g.g_end - g.g_begin;
  p.n_tiles = (p.n_groups + G - 1) / G;
  p.fixed_or = g.fixed_or;
  p.n_masks = g.n_masks;
  for (int i = 0; i < g.n_masks; ++i) p.masks[i] = g.masks[i];
  for (int j = 0; j < (1 << KS); ++j) p.off[j] = g.off[j];
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

// ------------------------------------------------------------------ entry
template <typename Real>
int launch_gate_impl(const GateLaunch& g, cudaStream_t s, int num_sms) {
  constexpr int DM = PrecisionTraits<Real>::kDirectMax;
  int klass = g.klass;
  if (klass == 0) return 0;
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

template <typename Real>
const char* kernel_name_impl(const GateLaunch& g) {
  constexpr int DM = PrecisionTraits<Real>::kDirectMax;
  int klass = g.klass;
  if (klass == 1 && !g.full_range) klass = g.ks <= DM ? 2 : 3;
  if (klass == 2 && g.ks > DM) klass = 3;
  switch (klass) {
    case 0: return "none";
    case 1: return "k_diag";
    case 2: return g.sparse ? "k_direct<sparse>" : "k_direct<dense>";
    default: return "k_tile";
  }
}

}  // namespace tsg
