// Device runtime of the B200 path and its C ABI (tsg_*): contexts, device
// statevectors, transfers, measurement reductions, kernel plans and
// programs (a planned fused circuit replayed as a CUDA graph).
//
// Reference operations replaced: Statevector / init_zero_state
// :505-524, plan_kernel :450, apply_kernel :459, run_circuit :525-533,
// compare_states :534, norm :543.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../host/handles.hpp"
#include "gate_launch.hpp"
#include "pass_jit.hpp"
#include "tilesim/pass.hpp"
#include "tilesim/plan.hpp"

using namespace tilesim;
using tsg_detail::require;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw SimError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

std::atomic<uint64_t> g_state_serial{1};

// ------------------------------------------------------------ reductions
constexpr int kRedThreads = 256;

template <typename Real>
__global__ void __launch_bounds__(kRedThreads) k_sumsq(const Real* __restrict__ re, const Real* __restrict__ im,
                                                         uint64_t n, double* __restrict__ partial) {
  double acc = 0.0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = re[i], y = im[i];
    acc = fma(x, x, fma(y, y, acc));
  }
  __shared__ double red[kRedThreads / 32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < kRedThreads / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
  }
}

// max_i |a_i - b_i| with b either a device state of type RealB or fp64 host data
template <typename RealA, typename RealB>
__global__ void __launch_bounds__(kRedThreads) k_maxdiff(const RealA* __restrict__ ar, const RealA* __restrict__ ai,
                                                           const RealB* __restrict__ br, const RealB* __restrict__ bi,
                                                           uint64_t n, double* __restrict__ partial) {
  double m = 0.0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double dr = static_cast<double>(ar[i]) - static_cast<double>(br[i]);
    const double di = static_cast<double>(ai[i]) - static_cast<double>(bi[i]);
    m = fmax(m, sqrt(dr * dr + di * di));
  }
  __shared__ double red[kRedThreads / 32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < kRedThreads / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) partial[blockIdx.x] = fmax(partial[blockIdx.x], m);
  }
}

// sum conj(a_i) b_i
template <typename Real>
__global__ void __launch_bounds__(kRedThreads) k_overlap(const Real* __restrict__ ar, const Real* __restrict__ ai,
                                                           const Real* __restrict__ br, const Real* __restrict__ bi,
                                                           uint64_t n, double* __restrict__ partial) {
  double sr = 0.0, si = 0.0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double xr = ar[i], xi = ai[i], yr = br[i], yi = bi[i];
    sr = fma(xr, yr, fma(xi, yi, sr));
    si = fma(xr, yi, fma(-xi, yr, si));
  }
  __shared__ double red[2][kRedThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = sr;
    red[1][threadIdx.x >> 5] = si;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    sr = threadIdx.x < kRedThreads / 32 ? red[0][threadIdx.x] : 0.0;
    si = threadIdx.x < kRedThreads / 32 ? red[1][threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      sr += __shfl_xor_sync(0xffffffffu, sr, o);
      si += __shfl_xor_sync(0xffffffffu, si, o);
    }
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = sr;
      partial[2 * blockIdx.x + 1] = si;
    }
  }
}

// ------------------------------------------------------- init / convert
// amplitudes at `count` indices into out[0, count) (re) and out[count, 2 count) (im)
template <typename Real>
__global__ void k_gather(const Real* re, const Real* im, const uint64_t* idx, uint64_t count, double* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count; i += uint64_t(gridDim.x) * blockDim.x) {
    out[i] = static_cast<double>(re[idx[i]]);
    out[count + i] = static_cast<double>(im[idx[i]]);
  }
}

template <typename Real>
__global__ void k_set_amp(Real* re, Real* im, uint64_t idx, double vr, double vi) {
  re[idx] = static_cast<Real>(vr);
  im[idx] = static_cast<Real>(vi);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// x_c(i) = u53(mix64(seed ^ ((2i + c) * golden))) - 0.5
template <typename Real>
__global__ void k_init_random(Real* re, Real* im, uint64_t n, uint64_t seed) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t a = mix64(seed ^ ((2 * i) * 0x9e3779b97f4a7c15ULL));
    const uint64_t b = mix64(seed ^ ((2 * i + 1) * 0x9e3779b97f4a7c15ULL));
    re[i] = static_cast<Real>(static_cast<double>(a >> 11) * 0x1.0p-53 - 0.5);
    im[i] = static_cast<Real>(static_cast<double>(b >> 11) * 0x1.0p-53 - 0.5);
  }
}

template <typename Real>
__global__ void k_scale(Real* re, Real* im, uint64_t n, double s) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    re[i] = static_cast<Real>(re[i] * s);
    im[i] = static_cast<Real>(im[i] * s);
  }
}

template <typename To, typename From>
__global__ void k_convert(To* __restrict__ dst, const From* __restrict__ src, uint64_t n) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = static_cast<To>(src[i]);
}

}  // namespace

// ============================================================== handles ===
struct tsg_ctx {
  int device = 0;
  int num_sms = 148;
  std::string name;
};

struct tsg_state {
  tsg_ctx* ctx = nullptr;
  int n = 0;
  int prec = 64;
  uint64_t serial = 0;
  void* re = nullptr;
  void* im = nullptr;
  cudaStream_t stream = nullptr;
  double* partial = nullptr;  // reduction scratch (2 * kMaxBlocks doubles)
  double* stage = nullptr;    // 2 x kStage doubles of transfer / compare staging
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // tsg_timer_*
  uint64_t size() const { return uint64_t{1} << n; }
  size_t amp_bytes() const { return prec == 64 ? 8 : 4; }
};

struct tsg_plan {
  tsg_ctx* ctx = nullptr;
  KernelPlan plan;
  void* dev_mat = nullptr;  // tile matrix scratch (state precision), allocated on demand
  size_t dev_mat_bytes = 0;
};

namespace {

constexpr int kMaxBlocks = 148 * 8;
constexpr uint64_t kStage = uint64_t{1} << 22;  // doubles per staging half (32 MiB)

struct ProgramGate {
  KernelPlan plan;
  LaunchStructure ls;
  tsg::GateLaunch launch;  // re/im filled per run
  size_t mat_offset = 0;   // into the device arena (tile class)
  bool has_mat = false;
  // standalone launches of a block-decomposed gate (tilesim::split_blocks);
  // empty: `launch` applies the gate
  std::vector<LaunchStructure> sub_ls;
  std::vector<tsg::GateLaunch> subs;
  std::vector<size_t> sub_mat;  // arena offset, or SIZE_MAX without a device matrix
  int batch = -1;          // >= 0: first gate of diagonal batch `batch`
  bool in_batch = false;   // applied by an earlier gate's batch launch
};

struct ProgramBatch {
  tsg::DiagBatchLaunch launch;  // re/im/tables filled per run
  size_t table_offset = 0;      // into the device arena
};

struct ProgramPass {
  tsg::PassLaunch launch;  // re/im/blob filled per run
  size_t blob_offset = 0;  // into the device arena
  std::vector<int> gates;
  int layouts_smem = 0;     // register layouts loaded through shared memory
  int layouts_shuffle = 0;  // ... reached with warp shuffles
};

// A run of qubit-permutation gates as one qubit permutation of the state:
// one in-place k_permute sweep per involution (one, or two when the composed
// permutation is not an involution).
struct ProgramPermute {
  std::vector<std::vector<int>> invs;  // launch order
};

// One launch of a program: a single gate, a diagonal batch, a tile pass or a
// qubit permutation.
enum StepKind : int { kStepGate = 0, kStepBatch = 1, kStepPass = 2, kStepPermute = 3 };
struct ProgramStep {
  int kind = kStepGate;
  int gate = 0;   // first gate applied by the step
  int index = 0;  // batch / pass index
  int n_gates = 1;
};

}  // namespace

struct tsg_program {
  tsg_ctx* ctx = nullptr;
  int n = 0;
  int prec = 64;
  std::vector<ProgramGate> gates;
  std::vector<ProgramBatch> batches;
  std::vector<ProgramPass> passes;
  std::vector<ProgramPermute> permutes;
  std::vector<ProgramStep> steps;
  void* arena = nullptr;
  double planning_s = 0.0;
  uint64_t launches = 0, bytes = 0, touched_bytes = 0, total_ops = 0;
  struct Graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
  };
  std::map<std::pair<tsg_state*, uint64_t>, Graph> graphs;
  std::map<std::pair<tsg_state*, uint64_t>, int> uses;  // runs per state before a graph is captured
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

void use_device(tsg_ctx* ctx) { ck(cudaSetDevice(ctx->device), "cudaSetDevice"); }

unsigned red_grid(uint64_t n) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(kMaxBlocks, (n + kRedThreads - 1) / kRedThreads)));
}

unsigned ew_grid(const tsg_ctx* ctx, uint64_t n) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(ctx->num_sms) * 16, (n + 255) / 256)));
}

double fetch_sum(tsg_state* st, unsigned blocks) {
  std::vector<double> h(blocks);
  ck(cudaMemcpyAsync(h.data(), st->partial, blocks * sizeof(double), cudaMemcpyDeviceToHost, st->stream), "partials");
  ck(cudaStreamSynchronize(st->stream), "reduction sync");
  double sum = 0.0, comp = 0.0;  // Kahan over block partials
  for (double v : h) {
    const double y = v - comp, t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
  return sum;
}

double state_norm(tsg_state* st) {
  const unsigned g = red_grid(st->size());
  if (st->prec == 64)
    k_sumsq<double><<<g, kRedThreads, 0, st->stream>>>((double*)st->re, (double*)st->im, st->size(), st->partial);
  else
    k_sumsq<float><<<g, kRedThreads, 0, st->stream>>>((float*)st->re, (float*)st->im, st->size(), st->partial);
  ck(cudaGetLastError(), "k_sumsq");
  return std::sqrt(fetch_sum(st, g));
}

void choose_dmma_perm(tsg::GateLaunch& g, const LaunchStructure& ls);

// fill a GateLaunch from a plan's launch structure
tsg::GateLaunch make_launch(const KernelPlan& p, const LaunchStructure& ls) {
  tsg::GateLaunch g;
  g.klass = static_cast<int>(ls.klass);
  g.k = p.gate.k();
  g.ks = ls.ks;
  g.sparse = ls.sparse ? 1 : 0;
  g.n = p.n;
  g.n_masks = static_cast<int>(p.group_masks.masks.size());
  for (int i = 0; i < g.n_masks; ++i) g.masks[i] = p.group_masks.masks[i];
  g.fixed_or = ls.control_values;
  g.n_ctrl = static_cast<int>(ls.controls.size());
  for (int i = 0; i < g.n_ctrl; ++i) g.ctrl[i] = ls.controls[i];
  for (int i = 0; i < ls.ks; ++i) g.sub_targets[i] = ls.sub_targets[i];
  for (size_t j = 0; j < ls.offsets.size() && j < (1u << tsg::kMaxSub); ++j) g.off[j] = ls.offsets[j];
  g.m_re = ls.sub_re.data();
  g.m_im = ls.sub_im.data();
  g.g_begin = 0;
  g.g_end = uint64_t{1} << (p.n - p.gate.k());
  g.full_range = true;
  choose_dmma_perm(g, ls);
  return g;
}

// Device copy of the snapped sub-matrix for the shared-memory / DMMA kernels:
// [Mr | Mi | Mr + Mi], D x D each, row-major, FP64 for both state precisions
// (k_tile reads the first two blocks, k_stream_dmma / k_dmma_direct all
// three), rows and columns in the launch's element order (GateLaunch::perm).
std::vector<unsigned char> tile_matrix_bytes(const LaunchStructure& ls, const tsg::GateLaunch& g) {
  if (g.klass == 1 && ls.ks > tsg::kMaxSub) {  // wide diagonal (k_diag_wide): [diag re][diag im], fp64
    const size_t D = size_t{1} << ls.ks;
    std::vector<unsigned char> out(2 * D * sizeof(double));
    double* d = reinterpret_cast<double*>(out.data());
    for (size_t j = 0; j < D; ++j) {
      d[j] = ls.sub_re[j * D + j];
      d[D + j] = ls.sub_im[j * D + j];
    }
    return out;
  }
  const size_t dd = ls.sub_re.size();
  const int D = 1 << ls.ks;
  std::vector<unsigned char> out(3 * dd * sizeof(double));
  double* d = reinterpret_cast<double*>(out.data());
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      const size_t i = static_cast<size_t>(r) * D + c, e = static_cast<size_t>(g.perm[r]) * D + g.perm[c];
      d[i] = ls.sub_re[e];
      d[dd + i] = ls.sub_im[e];
      d[2 * dd + i] = ls.sub_re[e] + ls.sub_im[e];
    }
  return out;
}

// Element order of a launch: identity, except for full-range sub-gates of
// 3..5 qubits (the DMMA stream kernels), which take the qubit order with the
// fewest nonzero DMMA tiles (<= 5! orders; ties keep the sorted order).
// Block-diagonal and tensor-product zero structure then fills whole tiles.
void choose_dmma_perm(tsg::GateLaunch& g, const LaunchStructure& ls) {
  const int D = 1 << g.ks;
  for (int j = 0; j < (1 << tsg::kMaxSub); ++j) g.perm[j] = static_cast<uint8_t>(j < D ? j : 0);
  if (!g.full_range || (g.klass != 2 && g.klass != 3) || g.ks < 3 || g.ks > 5) return;
  static const bool disabled = std::getenv("TSG_NO_DMMA_PERM") != nullptr;
  if (disabled) return;
  // nonzero pattern of [Mr | Mi | Mr + Mi] as one column bitmask per row
  // (D <= 32); a tile (row block rb, k-step k) of an element order P is
  // nonzero when a row P[r] of the block has a nonzero among the columns
  // P[4k .. 4k+3] -- the count dmma_tiles takes, from masks
  uint32_t nz[3][32] = {};
  bool dense = true;
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      const size_t e = static_cast<size_t>(r) * D + c;
      const double v[3] = {ls.sub_re[e], ls.sub_im[e], ls.sub_re[e] + ls.sub_im[e]};
      for (int m = 0; m < 3; ++m) {
        nz[m][r] |= static_cast<uint32_t>(v[m] != 0.0) << c;
        dense = dense && v[m] != 0.0;
      }
    }
  if (dense) return;  // every order has every tile nonzero
  auto tiles = [&](const int* P, int bound) {
    int t = 0;
    for (int k = 0; k < D / 4; ++k) {
      const uint32_t cols = (1u << P[4 * k]) | (1u << P[4 * k + 1]) | (1u << P[4 * k + 2]) | (1u << P[4 * k + 3]);
      for (int m = 0; m < 3; ++m)
        for (int rb = 0; rb < D / 8; ++rb) {
          bool any = false;
          for (int r = 8 * rb; r < 8 * rb + 8 && !any; ++r) any = (nz[m][P[r]] & cols) != 0;
          t += any;
        }
      if (t >= bound) return t;  // cannot beat the best so far
    }
    return t;
  };
  int bits[5] = {0, 1, 2, 3, 4}, P[32], best[32];
  for (int j = 0; j < D; ++j) best[j] = j;
  int best_tiles = tiles(best, 1 << 30);
  // targets on qubits 0, 1, 2: the sorted order stores each 8-row block of
  // outputs as 64 contiguous bytes; only orders that keep those three bits
  // in place compete (RQC-30's sparse 5-qubit gate on qubits 0..4: 9.9 ms
  // reordered and sparse, 9.3 ms sorted and dense, dmma_perm_ab.txt)
  const bool low3 = g.sub_targets[0] == 0 && g.sub_targets[1] == 1 && g.sub_targets[2] == 2;
  do {
    if (low3 && (bits[0] != 0 || bits[1] != 1 || bits[2] != 2)) continue;
    for (int j = 0; j < D; ++j) {
      int x = 0;
      for (int b = 0; b < g.ks; ++b) x |= ((j >> b) & 1) << bits[b];
      P[j] = x;
    }
    const int t = tiles(P, best_tiles);
    if (t < best_tiles) {
      best_tiles = t;
      std::copy(P, P + D, best);
    }
  } while (std::next_permutation(bits, bits + g.ks));
  // A reordered launch pays only when the product then skips its zero tiles
  // (dmma_setup: sparse at >= 1/4 zero tiles); otherwise the dense product
  // runs either way and the sorted order keeps each 8-row block of outputs
  // contiguous -- RQC-30's 5-qubit gate on qubits 0..4 with 88 of 96 tiles
  // nonzero under its best order: 9.96 ms reordered, 7.7 ms sorted.
  const int total = 3 * (D / 8) * (D / 4);
  static const bool any_gain = std::getenv("TSG_DMMA_PERM_ANY") != nullptr;  // round-2 rule (A/B runs)
  if (!any_gain && 4 * (total - best_tiles) < total) return;
  for (int j = 0; j < D; ++j) g.perm[j] = static_cast<uint8_t>(best[j]);
}

bool needs_tile_matrix(const tsg::GateLaunch& g, int prec) {
  const int dm = prec == 64 ? 4 : 5;
  if (g.klass == 3) return true;
  if (g.klass == 2 && g.ks >= 3) return true;  // k_stream_dmma / k_dmma_direct / k_tile
  if (g.klass == 1 && g.ks > dm) return true;  // sub-range diagonal falls back to tile
  return false;
}

int launch(tsg_state* st, const tsg::GateLaunch& g) {
  return st->prec == 64 ? tsg::launch_gate_f64(g, st->stream, st->ctx->num_sms)
                        : tsg::launch_gate_f32(g, st->stream, st->ctx->num_sms);
}

double touched_fraction(const LaunchStructure& ls) {
  if (ls.klass == KernelClass::Identity) return 0.0;
  return std::ldexp(1.0, -static_cast<int>(ls.controls.size()));
}

void fill_info(const KernelPlan& p, const LaunchStructure& ls, tsg_plan_info* out) {
  out->k = p.gate.k();
  out->kernel_class = static_cast<int>(ls.klass);
  out->sub_k = ls.ks;
  out->n_controls = static_cast<int>(ls.controls.size());
  out->sparse = ls.sparse ? 1 : 0;
  out->op_count = p.profile.op_count;
  out->entry_ops = p.entry_ops.size();
  out->loop_count = uint64_t{1} << (p.n - p.gate.k());
  out->touched_fraction = touched_fraction(ls);
  out->batched = 0;
  for (size_t i = 0; i < ls.controls.size() && i < 12; ++i) out->controls[i] = ls.controls[i];
  for (int i = 0; i < ls.ks && i < 12; ++i) out->sub_targets[i] = ls.sub_targets[i];
}

void run_step(tsg_state* st, tsg_program* prog, const ProgramStep& step) {
  unsigned char* arena = static_cast<unsigned char*>(prog->arena);
  if (step.kind == kStepBatch) {
    tsg::DiagBatchLaunch b = prog->batches[step.index].launch;
    b.re = st->re;
    b.im = st->im;
    b.tables = reinterpret_cast<const double*>(arena + prog->batches[step.index].table_offset);
    st->prec == 64 ? tsg::launch_diag_batch_f64(b, st->stream, st->ctx->num_sms)
                   : tsg::launch_diag_batch_f32(b, st->stream, st->ctx->num_sms);
    return;
  }
  if (step.kind == kStepPermute) {
    for (const std::vector<int>& inv : prog->permutes[step.index].invs) {
      tsg::PermuteLaunch pl;
      pl.n = prog->n;
      pl.re = st->re;
      pl.im = st->im;
      for (int q = 0; q < prog->n; ++q) pl.p[q] = inv[q];
      st->prec == 64 ? tsg::launch_permute_f64(pl, st->stream, st->ctx->num_sms)
                     : tsg::launch_permute_f32(pl, st->stream, st->ctx->num_sms);
    }
    return;
  }
  if (step.kind == kStepPass) {
    tsg::PassLaunch pl = prog->passes[step.index].launch;
    pl.re = st->re;
    pl.im = st->im;
    pl.blob = arena + prog->passes[step.index].blob_offset;
    st->prec == 64 ? tsg::launch_pass_f64(pl, st->stream, st->ctx->num_sms)
                   : tsg::launch_pass_f32(pl, st->stream, st->ctx->num_sms);
    return;
  }
  const ProgramGate& pg = prog->gates[step.gate];
  if (!pg.subs.empty()) {
    for (size_t i = 0; i < pg.subs.size(); ++i) {
      tsg::GateLaunch g = pg.subs[i];
      g.re = st->re;
      g.im = st->im;
      if (pg.sub_mat[i] != SIZE_MAX) g.dev_mat = arena + pg.sub_mat[i];
      launch(st, g);
    }
    return;
  }
  tsg::GateLaunch g = pg.launch;
  g.re = st->re;
  g.im = st->im;
  if (pg.has_mat) g.dev_mat = arena + pg.mat_offset;
  launch(st, g);
}

// marks (profiling): one event before every gate index, the gates a step
// applies after its first one share the step's interval (zero-length marks).
void run_program(tsg_state* st, tsg_program* prog, std::vector<cudaEvent_t>* marks) {
  size_t cursor = 0;
  for (const ProgramStep& step : prog->steps) {
    if (marks)
      for (; cursor <= static_cast<size_t>(step.gate); ++cursor) ck(cudaEventRecord((*marks)[cursor], st->stream), "event");
    run_step(st, prog, step);
  }
  if (marks) {
    for (; cursor < prog->gates.size(); ++cursor) ck(cudaEventRecord((*marks)[cursor], st->stream), "event");
    ck(cudaEventRecord(marks->back(), st->stream), "event");
  }
}

// Group runs of consecutive diagonal gates into one streaming launch when
// that moves fewer bytes than launching them separately (a separate launch
// touches only its active slice: touched_fraction = 2^-controls).
void plan_diagonal_batches(tsg_program* prog, std::vector<unsigned char>& arena) {
  if (prog->n < 2) return;
  auto batchable = [&](const ProgramGate& g) {
    return g.ls.klass == KernelClass::Diagonal && g.ls.ks <= 6 && !g.has_mat;
  };
  size_t i = 0;
  while (i < prog->gates.size()) {
    if (!batchable(prog->gates[i])) {
      ++i;
      continue;
    }
    size_t j = i;
    int entries = 0;
    double touched = 0.0;
    while (j < prog->gates.size() && batchable(prog->gates[j]) && j - i < static_cast<size_t>(tsg::kMaxBatch) &&
           entries + (1 << prog->gates[j].ls.ks) <= tsg::kMaxBatchEntries) {
      entries += 1 << prog->gates[j].ls.ks;
      touched += touched_fraction(prog->gates[j].ls);
      ++j;
    }
    if (j - i >= 2 && touched > 1.0) {
      ProgramBatch pb;
      tsg::DiagBatchLaunch& b = pb.launch;
      b.n = prog->n;
      std::vector<double> tab;
      for (size_t q = i; q < j; ++q) {
        const LaunchStructure& ls = prog->gates[q].ls;
        const int g = b.n_gates++;
        for (int c : ls.controls) b.cmask[g] |= uint64_t{1} << c;
        b.cval[g] = ls.control_values;
        b.ks[g] = ls.ks;
        for (int t = 0; t < ls.ks; ++t) b.tq[g][t] = ls.sub_targets[t];
        b.toff[g] = static_cast<int>(tab.size() / 2);
        const int d = 1 << ls.ks;
        for (int e = 0; e < d; ++e) {
          tab.push_back(ls.sub_re[e * d + e]);
          tab.push_back(ls.sub_im[e * d + e]);
        }
        prog->gates[q].in_batch = q != i;
      }
      b.n_entries = static_cast<int>(tab.size() / 2);
      pb.table_offset = (arena.size() + 255) & ~size_t{255};
      arena.resize(pb.table_offset + tab.size() * sizeof(double));
      std::memcpy(arena.data() + pb.table_offset, tab.data(), tab.size() * sizeof(double));
      prog->gates[i].batch = static_cast<int>(prog->batches.size());
      prog->batches.push_back(pb);
    }
    i = j;
  }
}

// Device blob of one tile pass (layout: gate_launch.hpp, PassLaunch).
template <typename Real>
void append_real2(std::vector<unsigned char>& v, double re, double im) {
  const Real x[2] = {static_cast<Real>(re), static_cast<Real>(im)};
  const unsigned char* b = reinterpret_cast<const unsigned char*>(x);
  v.insert(v.end(), b, b + sizeof x);
}

void pad16(std::vector<unsigned char>& v) { v.resize((v.size() + 15) & ~size_t{15}, 0); }

template <typename T>
void append_pod(std::vector<unsigned char>& v, const T& x) {
  const unsigned char* b = reinterpret_cast<const unsigned char*>(&x);
  v.insert(v.end(), b, b + sizeof(T));
}

// Tile-pass op records (layout: gate_launch.hpp).  A pass is built by
// walking its gates with the register layout the kernel will have: `pos`
// maps a qubit to its tile coordinate (-1 outside the tile) and `P` lists the
// r register positions (ascending) of the current layout; every other tile
// position is a thread position (thread-id bit b = b-th of them, ascending).
// Offsets are relative to the start of `data` and rebased by build_pass.
struct PassGeom {
  int M = 0, L = 0, r = 0;
  std::vector<int> pos;  // qubit -> tile coordinate
  std::vector<int> P;    // register positions of the current layout
  int reg_bit(int p) const {
    for (int k = 0; k < r; ++k)
      if (P[k] == p) return k;
    return -1;
  }
  // thread-id bit b -> tile position: the non-register positions, lanes
  // (bits 0-4) first; set by build_layout_op for each layout
  std::vector<int> tpos;
  int thread_bit(int p) const {
    for (size_t b = 0; b < tpos.size(); ++b)
      if (tpos[b] == p) return static_cast<int>(b);
    return -1;
  }
};

template <typename Real>
int padded_offset(uint32_t x, int L) {
  const int stride = (1 << L) + tsg::kPassPadBytes / static_cast<int>(sizeof(Real));
  return static_cast<int>((x >> L) * static_cast<uint32_t>(stride) + (x & ((1u << L) - 1)));
}

tsg::PassOp blank_op(int kind) {
  tsg::PassOp op;
  std::memset(&op, 0, sizeof op);
  op.kind = kind;
  return op;
}

// Shared-memory wavefronts of one register <-> tile move of a warp whose
// lanes sit on tile positions lanes[0..4] (scalar moves; 8-byte elements
// take at least 2)
template <typename Real>
int layout_wavefronts(const int* lanes, int L) {
  int words[32] = {0}, worst = 0;
  for (uint32_t l = 0; l < 32; ++l) {
    uint32_t x = 0;
    for (int b = 0; b < 5; ++b) x |= ((l >> b) & 1u) << lanes[b];
    const uint32_t w = static_cast<uint32_t>(padded_offset<Real>(x, L)) * (sizeof(Real) / 4);
    for (uint32_t k = 0; k < sizeof(Real) / 4; ++k) worst = std::max(worst, ++words[(w + k) % 32]);
  }
  return worst;
}

// LAYOUT op for g.P / g.tpos as set by the caller (tpos: thread-id bit ->
// tile position, lanes first).  n_swap > 0: the kernel reaches it from the
// previous layout with register <-> lane swaps (warp shuffles).
template <typename Real>
tsg::PassOp build_layout_op(PassGeom& g, std::vector<unsigned char>& data, int n_swap = 0, const int* swap_k = nullptr,
                            const int* swap_l = nullptr) {
  tsg::PassOp op = blank_op(tsg::kPassLayout);
  if (g.r + 1 > 6) throw SimError("pass: too many register positions");
  if (static_cast<int>(g.tpos.size()) != tsg::kPassLogThreads) throw SimError("pass: thread positions");
  op.n_swap = n_swap;
  for (int q = 0; q < n_swap; ++q) {
    op.swap_k[q] = static_cast<uint8_t>(swap_k[q]);
    op.swap_l[q] = static_cast<uint8_t>(swap_l[q]);
  }
  // per-thread tile coordinate of the thread part, looked up instead of
  // recomputed every tile
  pad16(data);
  op.aux_off = static_cast<int32_t>(data.size());
  for (uint32_t t = 0; t < static_cast<uint32_t>(tsg::kPassThreads); ++t) {
    uint32_t x = 0;
    for (size_t b = 0; b < g.tpos.size(); ++b) x |= ((t >> b) & 1u) << g.tpos[b];
    append_pod(data, x);
  }
  for (int k = 0; k < g.r; ++k) op.dep[k] = static_cast<uint32_t>(padded_offset<Real>(1u << g.P[k], g.L));
  // vector width of the register <-> shared-memory moves: register positions
  // 0, 1, .. = tile positions 0, 1, .. keep 2^vb registers in one 16-byte unit
  // (complex64 only: HES-30 pass 32.3 -> 24.2 ms; the kernel keeps scalar
  // moves for complex128, where pairs measured no faster)
  const int vmax = sizeof(Real) == 4 ? 2 : 0;
  int vb = 0;
  while (vb < vmax && vb < g.r && g.P[vb] == vb) ++vb;
  op.ks = vb;
  if (std::getenv("TSG_PASS_DEBUG")) {
    std::fprintf(stderr, "  layout%s P={", n_swap ? " (shuffles)" : "");
    for (int p : g.P) std::fprintf(stderr, " %d", p);
    std::fprintf(stderr, " } lanes={");
    for (int b = 0; b < 5; ++b) std::fprintf(stderr, " %d", g.tpos[b]);
    std::fprintf(stderr, " } warps={");
    for (int b = 5; b < tsg::kPassLogThreads; ++b) std::fprintf(stderr, " %d", g.tpos[b]);
    std::fprintf(stderr, " } wavefronts/move %d\n", layout_wavefronts<Real>(g.tpos.data(), g.L));
  }
  return op;
}

// Shared-memory cost (wavefronts per warp) of moving a layout's registers
// of both arrays once, as regs_to_smem / smem_to_regs do: complex64 layouts
// whose lowest register positions are tile positions 0, 1 move 2^vb
// registers per 16-byte-or-narrower vector access (build_layout_op's vb).
template <typename Real>
double layout_move_cost(const std::vector<int>& P, const int* lanes, int L) {
  const int R = 1 << static_cast<int>(P.size());
  int vb = 0;
  if (sizeof(Real) == 4)
    while (vb < 2 && vb < static_cast<int>(P.size()) && P[vb] == vb) ++vb;
  const uint32_t words = (sizeof(Real) / 4) << vb;  // 32-bit words per lane access
  int cnt[32] = {0}, worst = 0;
  for (uint32_t l = 0; l < 32; ++l) {
    uint32_t x = 0;
    for (int b = 0; b < 5; ++b) x |= ((l >> b) & 1u) << lanes[b];
    const uint32_t w = static_cast<uint32_t>(padded_offset<Real>(x, L)) * (sizeof(Real) / 4);
    for (uint32_t k = 0; k < words; ++k) worst = std::max(worst, ++cnt[(w + k) % 32]);
  }
  return 2.0 * (R >> vb) * worst;
}

// Widest layout change done with shuffles: complex64 changes of two and more
// bits measured slower than the shared-memory round trip (HES-30's block
// pass 25.1 -> 27.0 ms; the selects around each SHFL cost issue slots),
// complex128 one- and two-bit changes faster (QFT-30 73.5 -> 72.3 ms).
template <typename Real>
constexpr int shuffle_max_bits() {
  return sizeof(Real) == 8 ? 2 : 1;
}

// Thread positions for a layout loaded through shared memory with register
// positions P: 5 lanes + 3 warp positions out of the others.  A warp owns
// the amplitudes its lanes and registers span, so a later layout whose
// register positions avoid the warp positions is reached with warp shuffles
// (register <-> lane swaps: no shared-memory round trip, no barrier).  The
// lanes then drift onto other positions, and a later store of the registers
// (the end of the tile, a shared-memory op, the next shared-memory layout)
// pays the bank conflicts of where they are.  Cost model in shared-memory
// wavefronts per warp (layout_move_cost; a barrier ~32; a shuffle change of
// m bits 3 m R per 32-bit word of an element: a SHFL and the selects around
// it per pair member, issue slots rather than wavefronts -- measured: two-
// and three-bit changes of complex64 layouts ran slower than the shared-memory
// round trip they replaced): this load, the shuffles and the store after the last of
// them, against the default (sorted registers, lanes on the lowest free
// positions, every change a store and a load through shared memory).  Picks the warp
// positions and the number of the following register-current layouts
// (`next`) to reach with shuffles that save the most; *n_shuffle = 0 and the
// default when nothing is saved.  The simulated swaps are set_layout's.
template <typename Real>
std::vector<int> pick_thread_positions(const PassGeom& g, const std::vector<int>& P,
                                       const std::vector<std::vector<int>>& next, int* n_shuffle) {
  *n_shuffle = 0;
  auto default_lanes = [&](const std::vector<int>& regs) {
    std::vector<int> f;
    for (int p = 0; p < g.M; ++p)
      if (std::find(regs.begin(), regs.end(), p) == regs.end()) f.push_back(p);
    return f;
  };
  const std::vector<int> free_pos = default_lanes(P);
  if (static_cast<int>(free_pos.size()) != tsg::kPassLogThreads) throw SimError("pass: thread positions");
  std::vector<int> best = free_pos;  // lanes on the lowest free positions
  const char* shfl_env = std::getenv("TSG_PASS_SHFL");  // "0": every layout through shared memory
  if ((shfl_env && std::string(shfl_env) == "0") || next.empty()) return best;
  auto default_cost = [&](std::vector<int> regs) {
    std::sort(regs.begin(), regs.end());
    return layout_move_cost<Real>(regs, default_lanes(regs).data(), g.L);
  };
  const double R = static_cast<double>(1 << g.r), words = sizeof(Real) / 4;
  double best_gain = 0.0;
  const int nf = static_cast<int>(free_pos.size());
  for (int a = 0; a < nf; ++a)
    for (int b = a + 1; b < nf; ++b)
      for (int c = b + 1; c < nf; ++c) {
        const int W[3] = {free_pos[a], free_pos[b], free_pos[c]};
        auto in_w = [&](int p) { return p == W[0] || p == W[1] || p == W[2]; };
        std::vector<int> lanes;
        for (int p : free_pos)
          if (!in_w(p)) lanes.push_back(p);
        std::vector<int> cur = P;
        // this load against the default one
        double gain = default_cost(cur) - layout_move_cost<Real>(cur, lanes.data(), g.L);
        double best_here = -1e30;
        int best_len = 0;
        for (int j = 0; j <= static_cast<int>(next.size()); ++j) {
          // stop after j shuffle changes: the next store sees these lanes
          const double total = gain - (layout_move_cost<Real>(cur, lanes.data(), g.L) - default_cost(cur));
          if (total > best_here) {
            best_here = total;
            best_len = j;
          }
          if (j == static_cast<int>(next.size())) break;
          const std::vector<int>& Pn = next[j];
          bool ok = true;
          for (int p : Pn) ok = ok && !in_w(p);
          if (!ok) break;
          std::vector<int> out, in;
          for (int p : cur)
            if (std::find(Pn.begin(), Pn.end(), p) == Pn.end()) out.push_back(p);
          for (int p : Pn)
            if (std::find(cur.begin(), cur.end(), p) == cur.end()) in.push_back(p);
          if (static_cast<int>(in.size()) > shuffle_max_bits<Real>()) break;
          // the shared-memory change it replaces (default layouts on both sides)
          gain += default_cost(cur) + default_cost(Pn) + 32.0 - 3.0 * static_cast<double>(in.size()) * R * words;
          for (size_t q = 0; q < in.size(); ++q) {
            *std::find(lanes.begin(), lanes.end(), in[q]) = out[q];
            *std::find(cur.begin(), cur.end(), out[q]) = in[q];
          }
        }
        if (best_len > 0 && best_here > best_gain) {
          best_gain = best_here;
          *n_shuffle = best_len;
          best.clear();
          for (int p : free_pos)
            if (!in_w(p)) best.push_back(p);
          best.insert(best.end(), W, W + 3);
        }
      }
  return best;
}

// out-of-tile controls into cout, the rest returned as (tile position, value)
std::vector<std::pair<int, uint32_t>> split_controls(const LaunchStructure& ls, const PassGeom& g, tsg::PassOp& op) {
  std::vector<std::pair<int, uint32_t>> cin;
  for (int c : ls.controls) {
    const uint32_t v = static_cast<uint32_t>((ls.control_values >> c) & 1u);
    if (g.pos[c] < 0) {
      op.cout_mask |= uint64_t{1} << c;
      op.cout_val |= static_cast<uint64_t>(v) << c;
    } else {
      cin.emplace_back(g.pos[c], v);
    }
  }
  return cin;
}

template <typename Real>
tsg::PassOp build_diag_op(const LaunchStructure& ls, const PassGeom& g, std::vector<unsigned char>& data) {
  if (ls.ks > 7) throw SimError("pass: diagonal op wider than 7 qubits");
  tsg::PassOp op = blank_op(tsg::kPassDiagT);
  const int d = 1 << ls.ks;
  pad16(data);
  op.data_off = static_cast<int32_t>(data.size());
  op.ks = ls.ks;
  uint32_t thr_ctl_mask = 0, thr_ctl_val = 0;
  std::vector<std::pair<int, int>> thr_bits;  // (thread-id bit, table bit)
  bool on_thread = false, on_reg = false;
  for (const auto& [p, v] : split_controls(ls, g, op)) {
    const int k = g.reg_bit(p);
    if (k >= 0) {
      op.ictl_mask |= 1u << k;
      op.ictl_val |= v << k;
      on_reg = true;
    } else {
      const int tb = g.thread_bit(p);
      thr_ctl_mask |= 1u << tb;
      thr_ctl_val |= v << tb;
      on_thread = true;
    }
  }
  for (int b = 0; b < ls.ks; ++b) {
    const int q = ls.sub_targets[b], p = g.pos[q];
    if (p < 0) {
      op.out_gbit[op.n_out] = static_cast<uint8_t>(q);
      op.out_jbit[op.n_out++] = static_cast<uint8_t>(b);
    } else if (g.reg_bit(p) >= 0) {
      op.dep[g.reg_bit(p)] |= 1u << b;
      on_reg = true;
    } else {
      thr_bits.emplace_back(g.thread_bit(p), b);
      on_thread = true;
    }
  }
  op.kind = on_thread && on_reg ? tsg::kPassDiagX : (on_reg ? tsg::kPassDiagI : tsg::kPassDiagT);
  for (int j = 0; j < d; ++j) append_real2<Real>(data, ls.sub_re[j * d + j], ls.sub_im[j * d + j]);
  append_real2<Real>(data, 1.0, 0.0);  // inactive controls
  if (op.kind != tsg::kPassDiagI) {
    pad16(data);
    op.aux_off = static_cast<int32_t>(data.size());
    for (int t = 0; t < tsg::kPassThreads; ++t) {
      uint32_t v = 0;
      for (const auto& [tb, b] : thr_bits) v |= ((static_cast<uint32_t>(t) >> tb) & 1u) << b;
      if ((static_cast<uint32_t>(t) & thr_ctl_mask) != thr_ctl_val) v = 0xffu;
      data.push_back(static_cast<unsigned char>(v));
    }
  }
  return op;
}

// in-tile positions a diagonal sub-gate reads (targets and controls), ascending
std::vector<int> diag_signature(const LaunchStructure& ls, const PassGeom& g) {
  std::vector<int> sig;
  for (int q : ls.sub_targets)
    if (g.pos[q] >= 0) sig.push_back(g.pos[q]);
  for (int c : ls.controls)
    if (g.pos[c] >= 0) sig.push_back(g.pos[c]);
  std::sort(sig.begin(), sig.end());
  return sig;
}

// member of a diagonal group over signature `sig`: table index bits from the
// tile base (out bits, tc) and from the signature index e (dep[k] per bit k)
template <typename Real>
tsg::PassOp build_member_op(const LaunchStructure& ls, const PassGeom& g, const std::vector<int>& sig,
                            std::vector<unsigned char>& data) {
  tsg::PassOp op = blank_op(tsg::kPassDMember);
  const int d = 1 << ls.ks;
  pad16(data);
  op.data_off = static_cast<int32_t>(data.size());
  op.ks = ls.ks;
  auto sig_bit = [&](int p) { return static_cast<int>(std::find(sig.begin(), sig.end(), p) - sig.begin()); };
  for (const auto& [p, v] : split_controls(ls, g, op)) {
    op.ictl_mask |= 1u << sig_bit(p);
    op.ictl_val |= v << sig_bit(p);
  }
  for (int b = 0; b < ls.ks; ++b) {
    const int q = ls.sub_targets[b], p = g.pos[q];
    if (p < 0) {
      op.out_gbit[op.n_out] = static_cast<uint8_t>(q);
      op.out_jbit[op.n_out++] = static_cast<uint8_t>(b);
    } else {
      op.dep[sig_bit(p)] |= 1u << b;
    }
  }
  for (int j = 0; j < d; ++j) append_real2<Real>(data, ls.sub_re[j * d + j], ls.sub_im[j * d + j]);
  return op;
}

// group header: thread table (signature-index bits from thread positions),
// dep[k] = signature-index bits of register bit k, data_off = table entry offset
tsg::PassOp build_group_op(const PassGeom& g, const std::vector<int>& sig, int members, int entry_off,
                           std::vector<unsigned char>& data) {
  tsg::PassOp op = blank_op(tsg::kPassDGroup);
  op.ks = static_cast<int32_t>(sig.size());
  op.log2_groups = members;
  op.data_off = entry_off;
  std::vector<std::pair<int, int>> thr;  // (thread-id bit, signature bit)
  for (int k = 0; k < static_cast<int>(sig.size()); ++k) {
    const int rb = g.reg_bit(sig[k]);
    if (rb >= 0) op.dep[rb] |= 1u << k;
    else thr.emplace_back(g.thread_bit(sig[k]), k);
  }
  pad16(data);
  op.aux_off = static_cast<int32_t>(data.size());
  for (int t = 0; t < tsg::kPassThreads; ++t) {
    uint32_t v = 0;
    for (const auto& [tb, k] : thr) v |= ((static_cast<uint32_t>(t) >> tb) & 1u) << k;
    data.push_back(static_cast<unsigned char>(v));
  }
  return op;
}

// mixed (E) and block (B) bits of a non-diagonal sub-gate and the block matrices
struct BlockForm {
  std::vector<int> ebits, bbits;
  int ke = 0, nb = 0, de = 1;
  bool perm = false;
  int full(const LaunchStructure& ls, int je, int jb) const {
    int r = 0;
    for (int b = 0; b < ke; ++b) r |= ((je >> b) & 1) << ebits[b];
    for (int b = 0; b < nb; ++b) r |= ((jb >> b) & 1) << bbits[b];
    return r;
  }
};

BlockForm block_form(const LaunchStructure& ls) {
  BlockForm f;
  f.ebits = mixed_bits(ls);
  for (int b = 0; b < ls.ks; ++b)
    if (std::find(f.ebits.begin(), f.ebits.end(), b) == f.ebits.end()) f.bbits.push_back(b);
  f.ke = static_cast<int>(f.ebits.size());
  f.nb = static_cast<int>(f.bbits.size());
  f.de = 1 << f.ke;
  f.perm = monomial(ls);
  return f;
}

// blocks at the current end of `data`: GEN (D*D + 1 entries each) or Perm
// (src[D] element indices, 16-byte block, val[D]); perm_src_padded: Perm src
// entries are padded smem offsets (SPerm) instead of element indices (RPerm)
template <typename Real>
void append_blocks(const LaunchStructure& ls, const BlockForm& f, std::vector<unsigned char>& data,
                   const std::vector<uint32_t>* soffs) {
  const int d = 1 << ls.ks, de = f.de;
  for (int jb = 0; jb < (1 << f.nb); ++jb) {
    if (f.perm) {
      std::vector<int> col(de, 0);
      for (int r = 0; r < de; ++r)
        for (int c = 0; c < de; ++c) {
          const int e = f.full(ls, r, jb) * d + f.full(ls, c, jb);
          if (ls.sub_re[e] != 0.0 || ls.sub_im[e] != 0.0) col[r] = c;
        }
      for (int r = 0; r < de; ++r) append_pod(data, soffs ? (*soffs)[col[r]] : static_cast<uint32_t>(col[r]));
      pad16(data);
      for (int r = 0; r < de; ++r) {
        const int e = f.full(ls, r, jb) * d + f.full(ls, col[r], jb);
        append_real2<Real>(data, ls.sub_re[e], ls.sub_im[e]);
      }
    } else {
      for (int r = 0; r < de; ++r)
        for (int c = 0; c < de; ++c) {
          const int e = f.full(ls, r, jb) * d + f.full(ls, c, jb);
          append_real2<Real>(data, ls.sub_re[e], ls.sub_im[e]);
        }
      append_real2<Real>(data, 0.0, 0.0);  // bank padding between blocks
    }
  }
}

// RGen / RPerm: every mixed qubit is a register position of the layout
template <typename Real>
tsg::PassOp build_reg_op(const LaunchStructure& ls, const PassGeom& g, std::vector<unsigned char>& data) {
  BlockForm f = block_form(ls);
  // the kernel's block element index takes the mixed register bits in
  // ascending register order (reg_gen: deposit into rmask); after shuffle
  // changes the register positions need not ascend with the qubits, so the
  // blocks are laid out in that order
  std::stable_sort(f.ebits.begin(), f.ebits.end(), [&](int a, int b) {
    return g.reg_bit(g.pos[ls.sub_targets[a]]) < g.reg_bit(g.pos[ls.sub_targets[b]]);
  });
  tsg::PassOp op = blank_op(f.perm ? tsg::kPassRPerm : tsg::kPassRGen);
  op.ks = f.ke;
  for (int b : f.ebits) {
    const int k = g.reg_bit(g.pos[ls.sub_targets[b]]);
    if (k < 0) throw SimError("pass: register op on a non-register qubit");
    op.rmask |= 1 << k;
  }
  for (const auto& [p, v] : split_controls(ls, g, op)) {
    const int k = g.reg_bit(p);
    if (k >= 0) {
      op.ictl_mask |= 1u << k;
      op.ictl_val |= v << k;
    } else {
      op.tctl_mask |= 1u << p;
      op.tctl_val |= v << p;
    }
  }
  for (int i = 0; i < f.nb; ++i) {
    const int q = ls.sub_targets[f.bbits[i]], p = g.pos[q];
    if (p < 0) {
      op.out_gbit[op.n_out] = static_cast<uint8_t>(q);
      op.out_jbit[op.n_out++] = static_cast<uint8_t>(i);
    } else if (g.reg_bit(p) >= 0) {
      op.dep[g.reg_bit(p)] |= 1u << i;
    } else {
      op.tb_pos[op.n_tb] = static_cast<uint8_t>(p);
      op.tb_jbit[op.n_tb++] = static_cast<uint8_t>(i);
    }
  }
  // per-thread table: this thread's block bits on thread positions, 0xff when
  // its controls on thread positions are inactive (one lookup per op and tile
  // instead of a loop over tb_pos)
  op.thr_off = -1;
  if (op.n_tb > 0 || op.tctl_mask != 0) {
    pad16(data);
    op.thr_off = static_cast<int32_t>(data.size());
    for (uint32_t t = 0; t < static_cast<uint32_t>(tsg::kPassThreads); ++t) {
      uint32_t x = 0;
      for (size_t b = 0; b < g.tpos.size(); ++b) x |= ((t >> b) & 1u) << g.tpos[b];
      uint32_t v = 0;
      for (int b = 0; b < op.n_tb; ++b) v |= ((x >> op.tb_pos[b]) & 1u) << op.tb_jbit[b];
      if ((x & op.tctl_mask) != op.tctl_val) v = 0xffu;
      data.push_back(static_cast<unsigned char>(v));
    }
  }
  pad16(data);
  op.data_off = static_cast<int32_t>(data.size());
  op.aux_off = op.data_off;
  append_blocks<Real>(ls, f, data, nullptr);
  return op;
}

// SGen / SPerm: through shared memory, one thread (or a row split) per group
template <typename Real>
tsg::PassOp build_smem_op(const LaunchStructure& ls, const PassGeom& g, std::vector<unsigned char>& data) {
  const BlockForm f = block_form(ls);
  tsg::PassOp op = blank_op(f.perm ? tsg::kPassSPerm : tsg::kPassSGen);
  op.ks = f.ke;
  const int de = f.de, M = g.M, L = g.L;
  std::vector<int> zpos;  // tile positions fixed within a group: mixed qubits + in-tile controls
  uint32_t cin_val = 0;
  for (const auto& [p, v] : split_controls(ls, g, op)) {
    zpos.push_back(p);
    cin_val |= v << p;
  }
  for (int b : f.ebits) {
    const int p = g.pos[ls.sub_targets[b]];
    if (p < 0) throw SimError("pass: mixed qubit outside the tile");
    zpos.push_back(p);
  }
  std::vector<std::pair<int, int>> blk_in;  // (tile position, block bit)
  for (int i = 0; i < f.nb; ++i) {
    const int q = ls.sub_targets[f.bbits[i]], p = g.pos[q];
    if (p < 0) {
      op.out_gbit[op.n_out] = static_cast<uint8_t>(q);
      op.out_jbit[op.n_out++] = static_cast<uint8_t>(i);
    } else {
      blk_in.emplace_back(p, i);
    }
  }
  std::sort(zpos.begin(), zpos.end());
  const int count = static_cast<int>(zpos.size());
  uint64_t gm[64];
  const int n_gm = tsg::insertion_masks(zpos.data(), count, M - count, gm);
  op.log2_groups = M - count;
  auto deposit = [&](uint32_t v) {
    uint64_t x = 0;
    for (int i = 0; i < n_gm; ++i) x += (v & gm[i]) << i;
    return static_cast<uint32_t>(x);
  };
  auto entry = [&](uint32_t x) {  // padded offset | block bits << 16 (additive over disjoint bits)
    uint32_t jb = 0;
    for (const auto& [p, i] : blk_in) jb |= ((x >> p) & 1u) << i;
    return static_cast<uint32_t>(padded_offset<Real>(x, L)) | (jb << 16);
  };
  pad16(data);
  op.data_off = static_cast<int32_t>(data.size());
  std::vector<uint32_t> soffs(de);
  for (int j = 0; j < de; ++j) {
    uint32_t x = 0;
    for (int b = 0; b < f.ke; ++b) x |= static_cast<uint32_t>((j >> b) & 1) << g.pos[ls.sub_targets[f.ebits[b]]];
    soffs[j] = static_cast<uint32_t>(padded_offset<Real>(x, L));
    append_pod(data, soffs[j]);
  }
  pad16(data);
  const uint32_t n_groups = 1u << op.log2_groups;
  int rsplit = 0;  // fewer groups than threads: split each group's rows over 2^rsplit threads
  while ((n_groups << (rsplit + 1)) <= static_cast<uint32_t>(tsg::kPassThreads) && (1 << (rsplit + 1)) <= std::min(de, 8))
    ++rsplit;
  op.log2_rsplit = rsplit;
  if (rsplit == 0 && (f.ke >= 5 || (f.ke == 4 && sizeof(Real) == 8)))
    throw SimError("pass: this op needs a row split");  // no kernel instance without one (pass_gen_split)
  for (uint32_t t = 0; t < static_cast<uint32_t>(tsg::kPassThreads); ++t) {
    const uint32_t gi = t & (n_groups - 1);
    append_pod(data, (t < (n_groups << rsplit)) ? entry(deposit(gi) | cin_val) : 0u);
  }
  const uint32_t n_k = std::max<uint32_t>(1, n_groups / tsg::kPassThreads);
  for (uint32_t k = 0; k < n_k; ++k) append_pod(data, k == 0 ? 0u : entry(deposit(k * tsg::kPassThreads)));
  pad16(data);
  op.aux_off = static_cast<int32_t>(data.size());
  append_blocks<Real>(ls, f, data, f.perm ? &soffs : nullptr);
  return op;
}

// Register positions for a layout that holds `need` (tile positions):
// then the next ops' needs while they fit, then high positions.
std::vector<int> choose_layout(const std::vector<int>& need, const std::vector<std::vector<int>>& upcoming, int r,
                               int M, int L) {
  std::vector<int> P = need;
  for (const auto& e : upcoming) {
    std::vector<int> u = P;
    for (int p : e)
      if (std::find(u.begin(), u.end(), p) == u.end()) u.push_back(p);
    if (static_cast<int>(u.size()) > r) break;
    P = u;
  }
  for (int p = M - 1; p >= L && static_cast<int>(P.size()) < r; --p)
    if (std::find(P.begin(), P.end(), p) == P.end()) P.push_back(p);
  for (int p = L - 1; p >= 0 && static_cast<int>(P.size()) < r; --p)
    if (std::find(P.begin(), P.end(), p) == P.end()) P.push_back(p);
  std::sort(P.begin(), P.end());
  return P;
}

// Device blob of one tile pass: LAYOUT, then the gates in program order --
// register ops when the mixed qubits fit the register positions (a new
// LAYOUT when they are not the current ones), shared-memory ops otherwise,
// and RUN headers before runs of diagonal gates ordered by class (diagonal
// gates commute).
template <typename Real>
ProgramPass build_pass(const tsg_program* prog, const PassStep& step, const PassConfig& cfg,
                       std::vector<unsigned char>& arena) {
  const int n = prog->n, L = cfg.run_log2, M = cfg.tile_log2;
  const int nh = M - L;
  if (static_cast<int>(step.high.size()) != nh) throw SimError("pass: high tile qubit count");
  PassGeom g;
  g.M = M;
  g.L = L;
  g.r = M - tsg::kPassLogThreads;
  g.pos.assign(n, -1);
  for (int q = 0; q < L; ++q) g.pos[q] = q;
  for (int h = 0; h < nh; ++h) g.pos[step.high[h]] = L + h;

  // mixed tile positions of every register-capable gate (in order)
  const size_t ng = step.gates.size();
  std::vector<std::vector<int>> mixed(ng);
  std::vector<bool> reg_ok(ng, false);
  for (size_t i = 0; i < ng; ++i) {
    const LaunchStructure& ls = prog->gates[step.gates[i]].ls;
    if (ls.klass == KernelClass::Diagonal) continue;
    for (int b : mixed_bits(ls)) mixed[i].push_back(g.pos[ls.sub_targets[b]]);
    reg_ok[i] = static_cast<int>(mixed[i].size()) <= std::min(g.r, 3);
  }
  auto upcoming = [&](size_t from) {
    std::vector<std::vector<int>> u;
    for (size_t i = from; i < ng; ++i)
      if (reg_ok[i]) u.push_back(mixed[i]);
    return u;
  };

  // The register layouts the op loop below will set, in order (layout 0 is
  // the first load from shared memory), and whether the registers hold the
  // tile when each later one is needed (not right after a shared-memory op)
  // -- the thread positions of a shared-memory layout are picked so that
  // the following register-current ones can be reached with warp shuffles.
  std::vector<std::vector<int>> lay_P;
  std::vector<bool> lay_regs;
  {
    size_t first = 0;
    while (first < ng && !reg_ok[first]) ++first;
    lay_P.push_back(first < ng ? choose_layout(mixed[first], upcoming(first + 1), g.r, M, L)
                               : choose_layout({}, {}, g.r, M, L));
    lay_regs.push_back(false);
    bool after_smem = false, pending_diag = false;
    for (size_t i = 0; i < ng; ++i) {
      const LaunchStructure& ls = prog->gates[step.gates[i]].ls;
      if (ls.klass == KernelClass::Diagonal) {
        pending_diag = true;
        continue;
      }
      if (pending_diag) after_smem = false;  // a RUN in between: the kernel reloaded the registers
      pending_diag = false;
      if (reg_ok[i]) {
        bool fits = true;
        for (int p : mixed[i]) fits = fits && std::find(lay_P.back().begin(), lay_P.back().end(), p) != lay_P.back().end();
        if (!fits) {
          lay_P.push_back(choose_layout(mixed[i], upcoming(i + 1), g.r, M, L));
          lay_regs.push_back(!after_smem);
        }
        after_smem = false;
      } else {
        after_smem = true;
      }
    }
  }
  size_t lay = 0;      // next layout
  int shuffle_left = 0;  // following layouts the current thread positions plan to reach with shuffles
  // the layouts after `e` that could follow it with shuffles (registers current)
  auto shuffle_chain = [&](size_t e) {
    std::vector<std::vector<int>> nx;
    for (size_t f = e + 1; f < lay_P.size() && lay_regs[f]; ++f) nx.push_back(lay_P[f]);
    return nx;
  };
  std::vector<tsg::PassOp> ops;
  std::vector<unsigned char> data;
  auto set_layout = [&](bool regs_current) {
    const std::vector<int>& Pn = lay_P[lay];
    if (regs_current && shuffle_left > 0) {
      // register positions that leave / enter; shuffles when every entering
      // one is a lane position now
      std::vector<int> out, in;
      for (int p : g.P)
        if (std::find(Pn.begin(), Pn.end(), p) == Pn.end()) out.push_back(p);
      for (int p : Pn)
        if (g.reg_bit(p) < 0) in.push_back(p);
      bool lanes = static_cast<int>(in.size()) <= shuffle_max_bits<Real>();
      for (int p : in) lanes = lanes && g.thread_bit(p) >= 0 && g.thread_bit(p) < 5;
      if (lanes && !in.empty()) {
        int sk[4], sl[4];
        for (size_t q = 0; q < in.size(); ++q) {
          sk[q] = g.reg_bit(out[q]);
          sl[q] = g.thread_bit(in[q]);
          g.P[sk[q]] = in[q];
          g.tpos[sl[q]] = out[q];
        }
        ops.push_back(build_layout_op<Real>(g, data, static_cast<int>(in.size()), sk, sl));
        ++lay;
        --shuffle_left;
        return;
      }
    }
    g.P = Pn;
    g.tpos = pick_thread_positions<Real>(g, g.P, shuffle_chain(lay), &shuffle_left);
    ops.push_back(build_layout_op<Real>(g, data));
    ++lay;
  };
  set_layout(false);
  std::vector<const LaunchStructure*> run;  // the open run of diagonal gates
  auto flush_run = [&]() {
    if (run.empty()) return;
    // groups: largest signatures first, each op into the first group whose
    // signature stays <= kPassMaxSig bits with it (entries within budget)
    std::vector<std::pair<std::vector<int>, const LaunchStructure*>> items;
    for (const LaunchStructure* ls : run) items.emplace_back(diag_signature(*ls, g), ls);
    std::stable_sort(items.begin(), items.end(),
                     [](const auto& a, const auto& b) { return a.first.size() > b.first.size(); });
    std::vector<std::vector<int>> gsig;
    std::vector<std::vector<const LaunchStructure*>> gmem;
    std::vector<const LaunchStructure*> rest;
    int entries = 0;
    for (const auto& [sig, ls] : items) {
      // thread-position-only ops keep the per-thread DiagT path (no barrier,
      // all threads in parallel); groups take the rest
      bool on_reg = false;
      for (int p : sig) on_reg = on_reg || g.reg_bit(p) >= 0;
      if (static_cast<int>(sig.size()) > tsg::kPassMaxSig || !on_reg) {
        rest.push_back(ls);
        continue;
      }
      int best = -1, best_growth = 1 << 30;
      for (size_t q = 0; q < gsig.size(); ++q) {
        std::vector<int> u = gsig[q];
        for (int p : sig)
          if (std::find(u.begin(), u.end(), p) == u.end()) u.push_back(p);
        const int growth = (1 << u.size()) - (1 << gsig[q].size());
        if (static_cast<int>(u.size()) <= tsg::kPassMaxSig && entries + growth <= tsg::kPassMaxGEntries &&
            growth < best_growth) {
          best = static_cast<int>(q);
          best_growth = growth;
        }
      }
      if (best < 0) {
        if (entries + (1 << sig.size()) > tsg::kPassMaxGEntries) {
          rest.push_back(ls);
          continue;
        }
        gsig.push_back(sig);
        gmem.push_back({});
        entries += 1 << sig.size();
        best = static_cast<int>(gsig.size()) - 1;
      } else {
        for (int p : sig)
          if (std::find(gsig[best].begin(), gsig[best].end(), p) == gsig[best].end()) gsig[best].push_back(p);
        std::sort(gsig[best].begin(), gsig[best].end());
        entries += best_growth;
      }
      gmem[best].push_back(ls);
    }
    std::vector<tsg::PassOp> tops, xops;  // per-op classes for the rest
    for (const LaunchStructure* ls : rest) {
      tsg::PassOp op = build_diag_op<Real>(*ls, g, data);
      (op.kind == tsg::kPassDiagT ? tops : xops).push_back(op);  // DiagI ops always fit a group (<= 4 bits)
      if (op.kind == tsg::kPassDiagI) throw SimError("pass: register-only diagonal op outside a group");
    }
    tsg::PassOp hdr = blank_op(tsg::kPassRun);
    hdr.ks = static_cast<int32_t>(gsig.size());
    hdr.log2_groups = static_cast<int32_t>(tops.size());
    hdr.log2_rsplit = static_cast<int32_t>(xops.size());
    ops.push_back(hdr);
    int entry_off = 0;
    for (size_t q = 0; q < gsig.size(); ++q) {
      ops.push_back(build_group_op(g, gsig[q], static_cast<int>(gmem[q].size()), entry_off, data));
      entry_off += 1 << gsig[q].size();
      for (const LaunchStructure* ls : gmem[q]) ops.push_back(build_member_op<Real>(*ls, g, gsig[q], data));
    }
    ops.insert(ops.end(), tops.begin(), tops.end());
    ops.insert(ops.end(), xops.begin(), xops.end());
    run.clear();
  };
  for (size_t i = 0; i < ng; ++i) {
    const LaunchStructure& ls = prog->gates[step.gates[i]].ls;
    if (ls.klass == KernelClass::Diagonal) {
      run.push_back(&ls);
      continue;
    }
    flush_run();
    if (reg_ok[i]) {
      bool fits = true;
      for (int p : mixed[i]) fits = fits && g.reg_bit(p) >= 0;
      if (!fits) {
        bool planned = lay < lay_P.size();
        for (int p : mixed[i])
          planned = planned && std::find(lay_P[lay].begin(), lay_P[lay].end(), p) != lay_P[lay].end();
        if (!planned) throw SimError("pass: layout plan out of step");
        const bool regs_current = !ops.empty() && ops.back().kind != tsg::kPassSGen && ops.back().kind != tsg::kPassSPerm;
        set_layout(regs_current);
      }
      ops.push_back(build_reg_op<Real>(ls, g, data));
    } else {
      ops.push_back(build_smem_op<Real>(ls, g, data));
    }
  }
  flush_run();

  if (ops.size() > static_cast<size_t>(tsg::kPassMaxOps)) throw SimError("pass: too many ops");
  if (std::getenv("TSG_PASS_DEBUG")) {
    int cnt[11] = {0};
    for (const tsg::PassOp& op : ops) ++cnt[op.kind];
    std::fprintf(stderr, "pass gates %zu high", step.gates.size());
    for (int h : step.high) std::fprintf(stderr, " %d", h);
    std::fprintf(stderr,
                 ": layouts %d runs %d groups %d (members %d) diagT %d diagX %d rgen %d rperm %d sgen %d sperm %d\n",
                 cnt[0], cnt[1], cnt[9], cnt[10], cnt[2], cnt[4], cnt[5], cnt[6], cnt[7], cnt[8]);
  }
  const size_t data_base = (size_t{8} << nh) + ops.size() * sizeof(tsg::PassOp);
  for (tsg::PassOp& op : ops) {
    if (op.kind == tsg::kPassRun) continue;
    if (op.kind == tsg::kPassLayout || op.kind == tsg::kPassDGroup) {
      op.aux_off += static_cast<int32_t>(data_base);
      continue;
    }
    op.data_off += static_cast<int32_t>(data_base);
    if (op.kind != tsg::kPassDiagI && op.kind != tsg::kPassDMember) op.aux_off += static_cast<int32_t>(data_base);
    if ((op.kind == tsg::kPassRGen || op.kind == tsg::kPassRPerm) && op.thr_off >= 0)
      op.thr_off += static_cast<int32_t>(data_base);
  }
  std::vector<unsigned char> blob;
  for (int r = 0; r < (1 << nh); ++r) {
    uint64_t o = 0;
    for (int h = 0; h < nh; ++h) o |= static_cast<uint64_t>((r >> h) & 1) << step.high[h];
    append_pod(blob, o);
  }
  const unsigned char* ob = reinterpret_cast<const unsigned char*>(ops.data());
  blob.insert(blob.end(), ob, ob + ops.size() * sizeof(tsg::PassOp));
  blob.insert(blob.end(), data.begin(), data.end());
  pad16(blob);
  if (blob.size() > static_cast<size_t>(tsg::kPassMaxBlob)) throw SimError("pass: blob exceeds shared-memory budget");
  if (std::getenv("TSG_PASS_DEBUG")) std::fprintf(stderr, "  blob %zu bytes, %zu ops\n", blob.size(), ops.size());

  ProgramPass pp;
  pp.gates = step.gates;
  for (const tsg::PassOp& op : ops)
    if (op.kind == tsg::kPassLayout) ++(op.n_swap > 0 ? pp.layouts_shuffle : pp.layouts_smem);
  tsg::PassLaunch& pl = pp.launch;
  pl.n = n;
  pl.tile_log2 = M;
  pl.run_log2 = L;
  for (int h = 0; h < nh; ++h) pl.high[h] = step.high[h];
  pl.n_ops = static_cast<int>(ops.size());
  pl.blob_bytes = static_cast<int>(blob.size());
  pp.blob_offset = (arena.size() + 255) & ~size_t{255};
  arena.resize(pp.blob_offset + blob.size());
  std::memcpy(arena.data() + pp.blob_offset, blob.data(), blob.size());
  return pp;
}

// Contiguous region L of the DMMA stream kernel's tiles (dmma_geometry): the
// low bits holding 2^log2g groups plus every target or control below them.
int dmma_region(std::vector<int> qubits, int log2g) {
  int L = log2g;
  for (;;) {
    int below = 0;
    for (int q : qubits) below += q < L;
    if (log2g + below == L) return L;
    L = log2g + below;
  }
}

// A block split pays (measured on RQC-30, scripts/pass_bench.py) for a 5-6
// qubit sub-gate with ONE block qubit -- two half-sweep launches of a one
// qubit smaller sub-gate -- unless that qubit falls inside the part's
// contiguous tile region, where the half launches run double-size tiles.
// Four quarter launches (two block qubits) measured slower than the DMMA
// kernel's own zero-tile skipping.
bool split_pays(const LaunchStructure& ls, const std::vector<LaunchStructure>& parts, int prec) {
  if (parts.size() != 2 || parts[0].ks != ls.ks - 1) return false;
  const int amps_log2 = prec == 64 ? 11 : 12;  // DShape tile of the DMMA kernel
  for (const LaunchStructure& p : parts) {
    std::vector<int> q = p.sub_targets;
    q.insert(q.end(), p.controls.begin(), p.controls.end());
    const int L = dmma_region(q, amps_log2 - p.ks);
    for (int c : p.controls)
      if (std::find(ls.controls.begin(), ls.controls.end(), c) == ls.controls.end() && c < L) return false;
  }
  return true;
}

// The qubit permutation a run of permutation gates applies, as involutions.
// Index bit q of the result comes from bit src[q] of the input (new[y] =
// old[Pi(y)], Pi moving bit q to src[q]).  Gate g (targets t, sigma) moves
// the bit at t[b] to t[sigma[b]].  A permutation that is not an involution
// is split cycle by cycle into I2 o I1 (reflections of each cycle), applied
// as the sweep with I2, then the sweep with I1.
ProgramPermute compose_permutation(const tsg_program* prog, const std::vector<int>& gates) {
  const int n = prog->n;
  std::vector<int> src(n);
  for (int q = 0; q < n; ++q) src[q] = q;
  for (int gi : gates) {
    const LaunchStructure& ls = prog->gates[gi].ls;
    std::vector<int> sigma;
    if (!qubit_permutation(ls, &sigma)) throw SimError("permutation step: gate is not a qubit permutation");
    std::vector<int> next = src;
    for (int b = 0; b < ls.ks; ++b) next[ls.sub_targets[sigma[b]]] = src[ls.sub_targets[b]];
    src = std::move(next);
  }
  ProgramPermute out;
  bool invol = true;
  for (int q = 0; q < n; ++q) invol &= src[src[q]] == q;
  if (invol) {
    out.invs.push_back(src);
    return out;
  }
  std::vector<int> i1(n), i2(n);
  std::vector<bool> seen(n, false);
  for (int q = 0; q < n; ++q) {
    if (seen[q]) continue;
    std::vector<int> cyc;
    for (int r = q; !seen[r]; r = src[r]) {
      seen[r] = true;
      cyc.push_back(r);
    }
    const int m = static_cast<int>(cyc.size());
    for (int k = 0; k < m; ++k) {
      i1[cyc[k]] = cyc[(m - k) % m];      // c_k -> c_{-k}
      i2[cyc[k]] = cyc[(m + 1 - k) % m];  // c_k -> c_{1-k}
    }
  }
  out.invs.push_back(i2);
  out.invs.push_back(i1);
  return out;
}

// Steps of a program: tile passes (tilesim/pass.hpp) when the state holds at
// least one tile, else per-gate launches with diagonal batches.
void plan_steps(tsg_program* prog, std::vector<unsigned char>& arena) {
  const PassConfig cfg = pass_config(prog->prec, prog->n);
  const bool use_pass = !std::getenv("TSG_NO_PASS") && prog->n >= cfg.tile_log2;
  if (use_pass) {
    std::vector<LaunchStructure> ls;
    ls.reserve(prog->gates.size());
    for (const ProgramGate& pg : prog->gates) ls.push_back(pg.ls);
    for (const PassStep& st : plan_passes(ls, prog->n, cfg)) {
      ProgramStep step;
      step.gate = st.gates.front();
      step.n_gates = static_cast<int>(st.gates.size());
      if (st.is_permute) {
        step.kind = kStepPermute;
        step.index = static_cast<int>(prog->permutes.size());
        prog->permutes.push_back(compose_permutation(prog, st.gates));
        for (size_t i = 1; i < st.gates.size(); ++i) prog->gates[st.gates[i]].in_batch = true;
      } else if (st.is_pass) {
        step.kind = kStepPass;
        step.index = static_cast<int>(prog->passes.size());
        prog->passes.push_back(prog->prec == 64 ? build_pass<double>(prog, st, cfg, arena)
                                                : build_pass<float>(prog, st, cfg, arena));
        for (size_t i = 0; i < st.gates.size(); ++i) {
          prog->gates[st.gates[i]].batch = i == 0 ? step.index : -1;
          prog->gates[st.gates[i]].in_batch = i != 0;
        }
      }
      prog->steps.push_back(step);
    }
    // standalone 5..6-qubit sub-gates with block qubits: one launch per block
    // (2^-|B| of the state each, 2^|E|-qubit sub-gates off the FP64 roof)
    if (!std::getenv("TSG_NO_BLOCK_SPLIT"))
      for (const ProgramStep& step : prog->steps) {
        if (step.kind != kStepGate) continue;
        ProgramGate& pg = prog->gates[step.gate];
        if (pg.ls.ks < 5) continue;
        std::vector<LaunchStructure> parts = split_blocks(pg.ls, prog->prec);
        if (!split_pays(pg.ls, parts, prog->prec)) continue;
        pg.sub_ls = std::move(parts);
        for (const LaunchStructure& sl : pg.sub_ls) {
          tsg::GateLaunch g = make_launch(pg.plan, sl);
          size_t off = SIZE_MAX;
          if (needs_tile_matrix(g, prog->prec)) {
            const auto bytes = tile_matrix_bytes(sl, g);
            off = (arena.size() + 255) & ~size_t{255};
            arena.resize(off + bytes.size());
            std::copy(bytes.begin(), bytes.end(), arena.begin() + off);
          }
          pg.subs.push_back(g);
          pg.sub_mat.push_back(off);
        }
        for (size_t i = 0; i < pg.subs.size(); ++i) {  // host matrices of the (now stable) parts
          pg.subs[i].m_re = pg.sub_ls[i].sub_re.data();
          pg.subs[i].m_im = pg.sub_ls[i].sub_im.data();
        }
      }
    return;
  }
  if (!std::getenv("TSG_NO_DIAG_BATCH")) plan_diagonal_batches(prog, arena);
  for (size_t i = 0; i < prog->gates.size(); ++i) {
    const ProgramGate& pg = prog->gates[i];
    if (pg.in_batch || pg.ls.klass == KernelClass::Identity) continue;
    ProgramStep step;
    step.gate = static_cast<int>(i);
    if (pg.batch >= 0) {
      step.kind = kStepBatch;
      step.index = pg.batch;
      step.n_gates = prog->batches[pg.batch].launch.n_gates;
    }
    prog->steps.push_back(step);
  }
}

// JIT-compile the program's tile passes (pass_jit.cu), every distinct op
// table once, in parallel; a pass whose compile fails keeps the interpreter.
void jit_passes(tsg_program* prog, const std::vector<unsigned char>& arena) {
  if (prog->passes.empty() || !tsg::pass_jit_enabled(prog->n)) return;
  const int runs = prog->prec == 64 ? (1 << (11 - 5)) : (1 << (12 - 6));
  std::vector<std::string> src(prog->passes.size()), name(prog->passes.size());
  for (size_t i = 0; i < prog->passes.size(); ++i) {
    const ProgramPass& pp = prog->passes[i];
    const auto* ops = reinterpret_cast<const tsg::PassOp*>(arena.data() + pp.blob_offset + runs * sizeof(uint64_t));
    src[i] = tsg::pass_jit_source(prog->prec, ops, pp.launch.n_ops, &name[i]);
  }
  std::vector<const void*> kern(prog->passes.size(), nullptr);
  std::vector<std::string> err(prog->passes.size());
  std::vector<std::thread> pool;
  for (size_t i = 0; i < prog->passes.size(); ++i)
    pool.emplace_back([&, i] {
      try {
        cudaSetDevice(prog->ctx->device);
        kern[i] = tsg::pass_jit_kernel(src[i], name[i]);
      } catch (const std::exception& e) {
        err[i] = e.what();
      }
    });
  for (std::thread& t : pool) t.join();
  for (size_t i = 0; i < prog->passes.size(); ++i) {
    prog->passes[i].launch.jit = kern[i];
    if (!kern[i]) {
      static std::once_flag warned;
      std::call_once(warned, [&] { std::fprintf(stderr, "tilesim: pass JIT unavailable, interpreting (%s)\n", err[i].c_str()); });
    }
  }
}

// The standalone complex128 DMMA launches with zero 8 x 4 tiles get a
// JIT-compiled product with those tiles compiled out (pass_jit.hpp
// dmma_jit_spec; skipped loads and DMMAs cost nothing, unlike the runtime
// predicates of the sparse variant).  device = false: compile into the disk
// cache only (no device).
// (distinct kernels once; targets[i] = index into the returned specs of the
// i-th JIT launch, with `launches` its GateLaunch)
std::vector<std::pair<std::string, std::string>> dmma_jit_specs(tsg_program* prog,
                                                                 std::vector<tsg::GateLaunch*>* launches,
                                                                 std::vector<size_t>* targets) {
  std::vector<std::pair<std::string, std::string>> specs;
  if (prog->prec != 64 || !tsg::dmma_jit_enabled(prog->n)) return specs;
  std::map<std::string, size_t> index;
  auto consider = [&](tsg::GateLaunch& g) {
    std::string src, name;
    if (!tsg::dmma_jit_spec(g, &src, &name)) return;
    auto it = index.find(name);
    if (it == index.end()) {
      it = index.emplace(name, specs.size()).first;
      specs.emplace_back(std::move(src), std::move(name));
    }
    if (launches) {
      launches->push_back(&g);
      targets->push_back(it->second);
    }
  };
  for (const ProgramStep& step : prog->steps) {
    if (step.kind != kStepGate) continue;
    ProgramGate& pg = prog->gates[step.gate];
    if (pg.subs.empty()) consider(pg.launch);
    else
      for (tsg::GateLaunch& g : pg.subs) consider(g);
  }
  return specs;
}

void jit_gates(tsg_program* prog) {
  std::vector<tsg::GateLaunch*> launches;
  std::vector<size_t> targets;
  const auto specs = dmma_jit_specs(prog, &launches, &targets);
  if (specs.empty()) return;
  std::vector<const void*> kern(specs.size(), nullptr);
  std::vector<std::string> err(specs.size());
  std::vector<std::thread> pool;
  for (size_t i = 0; i < specs.size(); ++i)
    pool.emplace_back([&, i] {
      try {
        cudaSetDevice(prog->ctx->device);
        kern[i] = tsg::pass_jit_kernel(specs[i].first, specs[i].second);
      } catch (const std::exception& e) {
        err[i] = e.what();
      }
    });
  for (std::thread& t : pool) t.join();
  for (size_t i = 0; i < launches.size(); ++i) launches[i]->jit = kern[targets[i]];  // null: the generic kernel
  for (size_t i = 0; i < specs.size(); ++i)
    if (!kern[i]) {
      static std::once_flag warned;
      std::call_once(warned, [&] { std::fprintf(stderr, "tilesim: DMMA JIT unavailable (%s)\n", err[i].c_str()); });
    }
}

// run_circuit's planning: plan every gate, group the launches into steps
// (tile passes, block splits), upload matrices and pass blobs once.
// host half: plans, steps, arena contents (no device work)
std::unique_ptr<tsg_program> plan_program(tsg_ctx* ctx, const Circuit& fused, double zero_tol, double one_tol,
                                          int precision_bits, std::vector<unsigned char>& arena);

std::unique_ptr<tsg_program> build_program(tsg_ctx* ctx, const Circuit& fused, double zero_tol, double one_tol,
                                           int precision_bits) {
  use_device(ctx);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<unsigned char> arena;
  auto prog = plan_program(ctx, fused, zero_tol, one_tol, precision_bits, arena);
  if (!arena.empty()) {
    ck(cudaMalloc(&prog->arena, arena.size()), "cudaMalloc program arena");
    ck(cudaMemcpy(prog->arena, arena.data(), arena.size(), cudaMemcpyHostToDevice), "program arena upload");
  }
  jit_passes(prog.get(), arena);
  jit_gates(prog.get());
  ck(cudaEventCreate(&prog->ev0), "event");
  ck(cudaEventCreate(&prog->ev1), "event");
  prog->planning_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return prog;
}

std::unique_ptr<tsg_program> plan_program(tsg_ctx* ctx, const Circuit& fused, double zero_tol, double one_tol,
                                          int precision_bits, std::vector<unsigned char>& arena) {
  auto prog = std::make_unique<tsg_program>();
  prog->ctx = ctx;
  prog->n = fused.n_qubits;
  prog->prec = precision_bits;
  const uint64_t amp = precision_bits == 64 ? 16 : 8;
  for (const Gate& g : fused.gates) {
    ProgramGate pg;
    pg.plan = plan_kernel(g, prog->n, 0, zero_tol, one_tol, false);
    pg.ls = precision_bits == 64 ? pg.plan.launch : derive_launch(pg.plan, nullptr, precision_bits);
    pg.launch = make_launch(pg.plan, pg.ls);
    if (needs_tile_matrix(pg.launch, precision_bits)) {
      const auto bytes = tile_matrix_bytes(pg.ls, pg.launch);
      pg.mat_offset = (arena.size() + 255) & ~size_t{255};
      arena.resize(pg.mat_offset + bytes.size());
      std::copy(bytes.begin(), bytes.end(), arena.begin() + pg.mat_offset);
      pg.has_mat = true;
    }
    prog->total_ops += pg.plan.profile.op_count;
    prog->gates.push_back(std::move(pg));
  }
  plan_steps(prog.get(), arena);
  for (const ProgramStep& step : prog->steps) {  // one launch per step (block splits: one per part)
    const ProgramGate& pg = prog->gates[step.gate];
    const bool split = step.kind == kStepGate && !pg.subs.empty();
    if (step.kind == kStepPermute) {
      const uint64_t sweeps = prog->permutes[step.index].invs.size();
      prog->launches += sweeps;
      prog->bytes += sweeps * 2 * (uint64_t{1} << prog->n) * amp;
      prog->touched_bytes += sweeps * 2 * (uint64_t{1} << prog->n) * amp;
      continue;
    }
    prog->launches += split ? pg.subs.size() : 1;
    prog->bytes += 2 * (uint64_t{1} << prog->n) * amp;
    double frac = step.kind != kStepGate ? 1.0 : touched_fraction(pg.ls);
    if (split) {
      frac = 0.0;
      for (const LaunchStructure& sl : pg.sub_ls) frac += touched_fraction(sl);
    }
    prog->touched_bytes += static_cast<uint64_t>(2.0 * std::ldexp(1.0, prog->n) * amp * frac);
  }
  // the host snapped matrices referenced by launch.m_re/m_im must follow the moved vectors
  for (ProgramGate& pg : prog->gates) {
    pg.launch.m_re = pg.ls.sub_re.data();
    pg.launch.m_im = pg.ls.sub_im.data();
  }
  return prog;
}

}  // namespace

// ================================================================ C ABI ===
extern "C" {

int tsc_pass_jit_precompile(const tsc_circuit* fused, int precision_bits, double zero_tol, double one_tol,
                            int* n_passes) {
  TSG_TRY({
    require(fused && n_passes, "null argument");
    require(precision_bits == 64 || precision_bits == 32, "precision_bits must be 64 or 32");
    std::vector<unsigned char> arena;
    auto prog = plan_program(nullptr, fused->c, zero_tol, one_tol, precision_bits, arena);
    const int runs = precision_bits == 64 ? (1 << (11 - 5)) : (1 << (12 - 6));
    std::vector<std::thread> pool;
    std::vector<std::string> err(prog->passes.size());
    for (size_t i = 0; i < prog->passes.size(); ++i)
      pool.emplace_back([&, i] {
        try {
          const ProgramPass& pp = prog->passes[i];
          const auto* ops = reinterpret_cast<const tsg::PassOp*>(arena.data() + pp.blob_offset + runs * sizeof(uint64_t));
          std::string name;
          const std::string src = tsg::pass_jit_source(precision_bits, ops, pp.launch.n_ops, &name);
          tsg::pass_jit_cubin(src, name);
        } catch (const std::exception& e) {
          err[i] = e.what();
        }
      });
    // the JIT DMMA products of the program's standalone gates as well
    const auto specs = dmma_jit_specs(prog.get(), nullptr, nullptr);
    std::vector<std::string> gerr(specs.size());
    for (size_t i = 0; i < specs.size(); ++i)
      pool.emplace_back([&, i] {
        try {
          tsg::pass_jit_cubin(specs[i].first, specs[i].second);
        } catch (const std::exception& e) {
          gerr[i] = e.what();
        }
      });
    for (std::thread& t : pool) t.join();
    for (const std::string& e : err)
      if (!e.empty()) throw SimError(e);
    for (const std::string& e : gerr)
      if (!e.empty()) throw SimError(e);
    *n_passes = static_cast<int>(prog->passes.size());
  })
}

int tsg_device_count(int* out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (out) *out = n;
  return TSG_OK;
}

int tsg_ctx_info(const tsg_ctx* ctx, int* device, int* num_sms) {
  TSG_TRY({
    require(ctx != nullptr, "null handle");
    if (device) *device = ctx->device;
    if (num_sms) *num_sms = ctx->num_sms;
  })
}

int tsg_ctx_create(int device, tsg_ctx** out) {
  TSG_TRY({
    require(out != nullptr, "null output handle");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      throw SimError("no CUDA device available: the tilesim-b200 path has no CPU fallback");
    }
    require(device >= 0 && device < count, "device index out of range");
    auto ctx = std::make_unique<tsg_ctx>();
    ctx->device = device;
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10) throw SimError(std::string("device ") + prop.name + " is not sm_100 class (B200 required)");
    ctx->num_sms = prop.multiProcessorCount;
    ctx->name = prop.name;
    *out = ctx.release();
  })
}

int tsg_ctx_destroy(tsg_ctx* ctx) {
  delete ctx;
  return TSG_OK;
}

int tsg_state_create(tsg_ctx* ctx, int n_qubits, int precision_bits, tsg_state** out) {
  TSG_TRY({
    require(ctx && out, "null argument");
    require(n_qubits >= 1 && n_qubits <= 40, "qubit count must be in [1, 40] for one device");
    require(precision_bits == 64 || precision_bits == 32, "precision_bits must be 64 or 32");
    use_device(ctx);
    auto st = std::make_unique<tsg_state>();
    st->ctx = ctx;
    st->n = n_qubits;
    st->prec = precision_bits;
    st->serial = g_state_serial++;
    const size_t bytes = st->size() * st->amp_bytes();
    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const size_t need = 2 * bytes + 2 * kStage * sizeof(double) + 2 * kMaxBlocks * sizeof(double);
    if (need > free_b)
      throw SimError("statevector allocation failed: need " + std::to_string(2 * bytes) + " bytes (2^" +
                     std::to_string(n_qubits + (precision_bits == 64 ? 4 : 3)) + ") plus staging, " +
                     std::to_string(free_b) + " free");
    ck(cudaMalloc(&st->re, bytes), "cudaMalloc re");
    ck(cudaMalloc(&st->im, bytes), "cudaMalloc im");
    ck(cudaMalloc(&st->partial, 2 * kMaxBlocks * sizeof(double)), "cudaMalloc partial");
    ck(cudaMalloc(&st->stage, 2 * kStage * sizeof(double)), "cudaMalloc stage");
    ck(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    *out = st.release();
  })
}

int tsg_state_destroy(tsg_state* st) {
  if (!st) return TSG_OK;
  cudaSetDevice(st->ctx->device);
  if (st->stream) cudaStreamSynchronize(st->stream);
  cudaFree(st->re);
  cudaFree(st->im);
  cudaFree(st->partial);
  cudaFree(st->stage);
  if (st->stream) cudaStreamDestroy(st->stream);
  if (st->t0) cudaEventDestroy(st->t0);
  if (st->t1) cudaEventDestroy(st->t1);
  delete st;
  return TSG_OK;
}

int tsg_state_info(const tsg_state* st, int* n_qubits, int* precision_bits) {
  TSG_TRY({
    require(st != nullptr, "null handle");
    if (n_qubits) *n_qubits = st->n;
    if (precision_bits) *precision_bits = st->prec;
  })
}

int tsg_state_init_basis(tsg_state* st, uint64_t index) {
  TSG_TRY({
    require(st != nullptr, "null handle");
    require(index < st->size(), "basis index out of range");
    use_device(st->ctx);
    const size_t bytes = st->size() * st->amp_bytes();
    ck(cudaMemsetAsync(st->re, 0, bytes, st->stream), "memset re");
    ck(cudaMemsetAsync(st->im, 0, bytes, st->stream), "memset im");
    if (st->prec == 64) k_set_amp<double><<<1, 1, 0, st->stream>>>((double*)st->re, (double*)st->im, index, 1.0, 0.0);
    else k_set_amp<float><<<1, 1, 0, st->stream>>>((float*)st->re, (float*)st->im, index, 1.0, 0.0);
    ck(cudaGetLastError(), "k_set_amp");
  })
}

int tsg_state_init_zero(tsg_state* st) { return tsg_state_init_basis(st, 0); }

int tsg_state_init_random(tsg_state* st, uint64_t seed) {
  TSG_TRY({
    require(st != nullptr, "null handle");
    use_device(st->ctx);
    const unsigned g = ew_grid(st->ctx, st->size());
    if (st->prec == 64) k_init_random<double><<<g, 256, 0, st->stream>>>((double*)st->re, (double*)st->im, st->size(), seed);
    else k_init_random<float><<<g, 256, 0, st->stream>>>((float*)st->re, (float*)st->im, st->size(), seed);
    ck(cudaGetLastError(), "k_init_random");
    const double nrm = state_norm(st);
    if (st->prec == 64) k_scale<double><<<g, 256, 0, st->stream>>>((double*)st->re, (double*)st->im, st->size(), 1.0 / nrm);
    else k_scale<float><<<g, 256, 0, st->stream>>>((float*)st->re, (float*)st->im, st->size(), 1.0 / nrm);
    ck(cudaGetLastError(), "k_scale");
  })
}

int tsg_state_upload_range(tsg_state* st, uint64_t begin, uint64_t count, const double* re, const double* im) {
  TSG_TRY({
    require(st && re && im, "null argument");
    require(begin <= st->size() && count <= st->size() - begin, "upload range outside the state");
    use_device(st->ctx);
    if (st->prec == 64) {
      ck(cudaMemcpyAsync((double*)st->re + begin, re, count * 8, cudaMemcpyHostToDevice, st->stream), "upload re");
      ck(cudaMemcpyAsync((double*)st->im + begin, im, count * 8, cudaMemcpyHostToDevice, st->stream), "upload im");
    } else {
      for (uint64_t b = 0; b < count; b += kStage) {
        const uint64_t c = std::min(kStage, count - b);
        ck(cudaMemcpyAsync(st->stage, re + b, c * 8, cudaMemcpyHostToDevice, st->stream), "upload re");
        ck(cudaMemcpyAsync(st->stage + kStage, im + b, c * 8, cudaMemcpyHostToDevice, st->stream), "upload im");
        k_convert<float, double><<<ew_grid(st->ctx, c), 256, 0, st->stream>>>((float*)st->re + begin + b, st->stage, c);
        k_convert<float, double><<<ew_grid(st->ctx, c), 256, 0, st->stream>>>((float*)st->im + begin + b,
                                                                             st->stage + kStage, c);
        ck(cudaGetLastError(), "k_convert");
      }
    }
    ck(cudaStreamSynchronize(st->stream), "upload sync");
  })
}

int tsg_state_upload(tsg_state* st, const double* re, const double* im) {
  if (!st) {
    tsg_detail::set_error("null handle");
    return TSG_ERR_CONFIG;
  }
  return tsg_state_upload_range(st, 0, st->size(), re, im);
}

int tsg_state_download_range(tsg_state* st, uint64_t begin, uint64_t count, double* re, double* im) {
  TSG_TRY({
    require(st && re && im, "null argument");
    require(begin <= st->size() && count <= st->size() - begin, "download range outside the state");
    use_device(st->ctx);
    if (st->prec == 64) {
      ck(cudaMemcpyAsync(re, (double*)st->re + begin, count * 8, cudaMemcpyDeviceToHost, st->stream), "download re");
      ck(cudaMemcpyAsync(im, (double*)st->im + begin, count * 8, cudaMemcpyDeviceToHost, st->stream), "download im");
    } else {
      for (uint64_t b = 0; b < count; b += kStage) {
        const uint64_t c = std::min(kStage, count - b);
        k_convert<double, float><<<ew_grid(st->ctx, c), 256, 0, st->stream>>>(st->stage, (float*)st->re + begin + b, c);
        k_convert<double, float><<<ew_grid(st->ctx, c), 256, 0, st->stream>>>(st->stage + kStage, (float*)st->im + begin + b, c);
        ck(cudaGetLastError(), "k_convert");
        ck(cudaMemcpyAsync(re + b, st->stage, c * 8, cudaMemcpyDeviceToHost, st->stream), "download re");
        ck(cudaMemcpyAsync(im + b, st->stage + kStage, c * 8, cudaMemcpyDeviceToHost, st->stream), "download im");
      }
    }
    ck(cudaStreamSynchronize(st->stream), "download sync");
  })
}

int tsg_state_gather(tsg_state* st, const uint64_t* indices, uint64_t count, double* re, double* im) {
  TSG_TRY({
    require(st && indices && re && im, "null argument");
    require(count <= kStage / 2, "gather: too many indices (at most half the staging buffer)");
    for (uint64_t i = 0; i < count; ++i) require(indices[i] < st->size(), "gather index outside the state");
    if (count == 0) return TSG_OK;
    use_device(st->ctx);
    // indices in the staging buffer's second half, values into its first 2 count doubles
    uint64_t* didx = reinterpret_cast<uint64_t*>(st->stage + kStage);
    ck(cudaMemcpyAsync(didx, indices, count * sizeof(uint64_t), cudaMemcpyHostToDevice, st->stream), "gather indices");
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((count + 255) / 256, 1024));
    if (st->prec == 64) k_gather<double><<<grid, 256, 0, st->stream>>>((double*)st->re, (double*)st->im, didx, count, st->stage);
    else k_gather<float><<<grid, 256, 0, st->stream>>>((float*)st->re, (float*)st->im, didx, count, st->stage);
    ck(cudaGetLastError(), "k_gather");
    std::vector<double> buf(2 * count);
    ck(cudaMemcpyAsync(buf.data(), st->stage, 2 * count * sizeof(double), cudaMemcpyDeviceToHost, st->stream), "gather");
    ck(cudaStreamSynchronize(st->stream), "gather sync");
    std::copy(buf.begin(), buf.begin() + count, re);
    std::copy(buf.begin() + count, buf.end(), im);
  })
}

int tsg_state_download(tsg_state* st, double* re, double* im) {
  if (!st) {
    tsg_detail::set_error("null handle");
    return TSG_ERR_CONFIG;
  }
  return tsg_state_download_range(st, 0, st->size(), re, im);
}

// QSV1 amplitude dump: 16-byte header ("QSV1", u8 precision
// bits 32|64, u8 n, 10 zero bytes), then re[2^n] and im[2^n] little-endian
// in the state's precision; streamed through a 64 MiB host buffer.
int tsg_state_dump(tsg_state* st, const char* path) {
  TSG_TRY({
    require(st && path, "null argument");
    use_device(st->ctx);
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), std::fclose);
    if (!f) throw SimError(std::string("cannot open ") + path + " for writing");
    unsigned char hdr[16] = {'Q', 'S', 'V', '1', static_cast<unsigned char>(st->prec), static_cast<unsigned char>(st->n)};
    if (std::fwrite(hdr, 1, 16, f.get()) != 16) throw SimError("QSV1 header write failed");
    ck(cudaStreamSynchronize(st->stream), "dump sync");
    const size_t total = st->size() * st->amp_bytes(), chunk = size_t{64} << 20;
    std::vector<unsigned char> buf(std::min(total, chunk));
    for (const void* arr : {st->re, st->im})
      for (size_t off = 0; off < total; off += chunk) {
        const size_t cnt = std::min(chunk, total - off);
        ck(cudaMemcpy(buf.data(), static_cast<const unsigned char*>(arr) + off, cnt, cudaMemcpyDeviceToHost), "dump copy");
        if (std::fwrite(buf.data(), 1, cnt, f.get()) != cnt) throw SimError("QSV1 write failed");
      }
  })
}

int tsg_state_load(tsg_state* st, const char* path) {
  TSG_TRY({
    require(st && path, "null argument");
    use_device(st->ctx);
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "rb"), std::fclose);
    if (!f) throw SimError(std::string("cannot open ") + path);
    unsigned char hdr[16];
    if (std::fread(hdr, 1, 16, f.get()) != 16 || std::memcmp(hdr, "QSV1", 4) != 0)
      throw ParseError(std::string(path) + ": not a QSV1 file");
    if (hdr[4] != st->prec || hdr[5] != st->n)
      throw ConfigError(std::string(path) + ": QSV1 precision / qubit count differ from the state");
    const size_t total = st->size() * st->amp_bytes(), chunk = size_t{64} << 20;
    std::vector<unsigned char> buf(std::min(total, chunk));
    ck(cudaStreamSynchronize(st->stream), "load sync");
    for (void* arr : {st->re, st->im})
      for (size_t off = 0; off < total; off += chunk) {
        const size_t cnt = std::min(chunk, total - off);
        if (std::fread(buf.data(), 1, cnt, f.get()) != cnt) throw ParseError(std::string(path) + ": truncated QSV1 data");
        ck(cudaMemcpy(static_cast<unsigned char*>(arr) + off, buf.data(), cnt, cudaMemcpyHostToDevice), "load copy");
      }
  })
}

int tsg_state_copy(tsg_state* dst, const tsg_state* src) {
  TSG_TRY({
    require(dst && src, "null argument");
    require(dst->n == src->n && dst->prec == src->prec, "state shapes differ");
    use_device(dst->ctx);
    ck(cudaStreamSynchronize(src->stream), "source sync");
    const size_t bytes = dst->size() * dst->amp_bytes();
    ck(cudaMemcpyAsync(dst->re, src->re, bytes, cudaMemcpyDeviceToDevice, dst->stream), "copy re");
    ck(cudaMemcpyAsync(dst->im, src->im, bytes, cudaMemcpyDeviceToDevice, dst->stream), "copy im");
  })
}

int tsg_synchronize(tsg_state* st) {
  TSG_TRY({
    require(st != nullptr, "null handle");
    ck(cudaStreamSynchronize(st->stream), "stream sync");
  })
}

int tsg_timer_begin(tsg_state* st) {
  TSG_TRY({
    require(st != nullptr, "null handle");
    use_device(st->ctx);
    if (!st->t0) ck(cudaEventCreate(&st->t0), "event");
    if (!st->t1) ck(cudaEventCreate(&st->t1), "event");
    ck(cudaEventRecord(st->t0, st->stream), "event record");
  })
}

int tsg_timer_end(tsg_state* st, double* seconds) {
  TSG_TRY({
    require(st && seconds && st->t0, "timer not started");
    ck(cudaEventRecord(st->t1, st->stream), "event record");
    ck(cudaEventSynchronize(st->t1), "event sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, st->t0, st->t1), "elapsed");
    *seconds = ms * 1e-3;
  })
}

int tsg_norm(tsg_state* st, double* out) {
  TSG_TRY({
    require(st && out, "null argument");
    use_device(st->ctx);
    *out = state_norm(st);
  })
}

int tsg_compare(tsg_state* st, const double* re, const double* im, double* maxdiff) {
  TSG_TRY({
    require(st && re && im && maxdiff, "null argument");
    use_device(st->ctx);
    const unsigned g = red_grid(kStage);
    ck(cudaMemsetAsync(st->partial, 0, g * sizeof(double), st->stream), "memset partial");
    for (uint64_t b = 0; b < st->size(); b += kStage) {
      const uint64_t c = std::min(kStage, st->size() - b);
      ck(cudaMemcpyAsync(st->stage, re + b, c * 8, cudaMemcpyHostToDevice, st->stream), "compare upload");
      ck(cudaMemcpyAsync(st->stage + kStage, im + b, c * 8, cudaMemcpyHostToDevice, st->stream), "compare upload");
      if (st->prec == 64)
        k_maxdiff<double, double><<<g, kRedThreads, 0, st->stream>>>((double*)st->re + b, (double*)st->im + b, st->stage,
                                                                   st->stage + kStage, c, st->partial);
      else
        k_maxdiff<float, double><<<g, kRedThreads, 0, st->stream>>>((float*)st->re + b, (float*)st->im + b, st->stage,
                                                                  st->stage + kStage, c, st->partial);
      ck(cudaGetLastError(), "k_maxdiff");
    }
    std::vector<double> h(g);
    ck(cudaMemcpyAsync(h.data(), st->partial, g * sizeof(double), cudaMemcpyDeviceToHost, st->stream), "partials");
    ck(cudaStreamSynchronize(st->stream), "compare sync");
    *maxdiff = *std::max_element(h.begin(), h.end());
  })
}

int tsg_compare_states(tsg_state* a, tsg_state* b, double* maxdiff) {
  TSG_TRY({
    require(a && b && maxdiff, "null argument");
    require(a->n == b->n, "state sizes differ");
    use_device(a->ctx);
    ck(cudaStreamSynchronize(b->stream), "sync b");
    const unsigned g = red_grid(a->size());
    ck(cudaMemsetAsync(a->partial, 0, g * sizeof(double), a->stream), "memset partial");
    if (a->prec == 64 && b->prec == 64)
      k_maxdiff<double, double><<<g, kRedThreads, 0, a->stream>>>((double*)a->re, (double*)a->im, (double*)b->re,
                                                                (double*)b->im, a->size(), a->partial);
    else if (a->prec == 32 && b->prec == 32)
      k_maxdiff<float, float><<<g, kRedThreads, 0, a->stream>>>((float*)a->re, (float*)a->im, (float*)b->re,
                                                              (float*)b->im, a->size(), a->partial);
    else if (a->prec == 32)
      k_maxdiff<float, double><<<g, kRedThreads, 0, a->stream>>>((float*)a->re, (float*)a->im, (double*)b->re,
                                                               (double*)b->im, a->size(), a->partial);
    else
      k_maxdiff<double, float><<<g, kRedThreads, 0, a->stream>>>((double*)a->re, (double*)a->im, (float*)b->re,
                                                               (float*)b->im, a->size(), a->partial);
    ck(cudaGetLastError(), "k_maxdiff");
    std::vector<double> h(g);
    ck(cudaMemcpyAsync(h.data(), a->partial, g * sizeof(double), cudaMemcpyDeviceToHost, a->stream), "partials");
    ck(cudaStreamSynchronize(a->stream), "compare sync");
    *maxdiff = *std::max_element(h.begin(), h.end());
  })
}

int tsg_overlap(tsg_state* a, tsg_state* b, double* re, double* im) {
  TSG_TRY({
    require(a && b && re && im, "null argument");
    require(a->n == b->n && a->prec == b->prec, "state shapes differ");
    use_device(a->ctx);
    ck(cudaStreamSynchronize(b->stream), "sync b");
    const unsigned g = red_grid(a->size());
    if (a->prec == 64)
      k_overlap<double><<<g, kRedThreads, 0, a->stream>>>((double*)a->re, (double*)a->im, (double*)b->re,
                                                          (double*)b->im, a->size(), a->partial);
    else
      k_overlap<float><<<g, kRedThreads, 0, a->stream>>>((float*)a->re, (float*)a->im, (float*)b->re, (float*)b->im,
                                                         a->size(), a->partial);
    ck(cudaGetLastError(), "k_overlap");
    std::vector<double> h(2 * g);
    ck(cudaMemcpyAsync(h.data(), a->partial, 2 * g * sizeof(double), cudaMemcpyDeviceToHost, a->stream), "partials");
    ck(cudaStreamSynchronize(a->stream), "overlap sync");
    double sr = 0, si = 0;
    for (unsigned i = 0; i < g; ++i) {
      sr += h[2 * i];
      si += h[2 * i + 1];
    }
    *re = sr;
    *im = si;
  })
}

// ------------------------------------------------------------------ plans
int tsg_plan_create(tsg_ctx* ctx, int n_qubits, int k, const int* targets, const double* matrix, double zero_tol,
                    double one_tol, int runtime_matrix, tsg_plan** out) {
  TSG_TRY({
    require(out && targets && matrix, "null argument");
    require(k >= 1 && k <= kFusedQubitCap, "gate size must be in [1, 12]");
    require(zero_tol >= 0 && one_tol >= 0, "tolerances must be >= 0");
    GateMatrix m(k);
    for (size_t i = 0; i < m.entries().size(); ++i) m.entries()[i] = cplx(matrix[2 * i], matrix[2 * i + 1]);
    Gate g = make_gate(std::move(m), std::vector<int>(targets, targets + k));
    auto p = std::make_unique<tsg_plan>();
    p->ctx = ctx;
    p->plan = plan_kernel(g, n_qubits, 0, zero_tol, one_tol, runtime_matrix != 0);
    *out = p.release();
  })
}

int tsg_plan_destroy(tsg_plan* p) {
  if (!p) return TSG_OK;
  if (p->dev_mat) cudaFree(p->dev_mat);
  delete p;
  return TSG_OK;
}

int tsg_plan_info_get(const tsg_plan* p, tsg_plan_info* out) {
  TSG_TRY({
    require(p && out, "null argument");
    fill_info(p->plan, p->plan.launch, out);
  })
}

int tsg_apply(tsg_state* st, const tsg_plan* pc, const double* matrix_override, uint64_t t_begin, uint64_t t_end) {
  TSG_TRY({
    require(st && pc, "null argument");
    tsg_plan* p = const_cast<tsg_plan*>(pc);
    const KernelPlan& kp = p->plan;
    if (kp.n != st->n) throw ConfigError("plan was made for a different qubit count");
    if (matrix_override && !kp.runtime_matrix) throw SimError("matrix override given for a plan with baked matrix");
    if (!matrix_override && kp.runtime_matrix) throw SimError("runtime-matrix plan needs a matrix override");
    const uint64_t groups = uint64_t{1} << (kp.n - kp.gate.k());
    if (t_end == UINT64_MAX) t_end = groups;
    if (t_begin > t_end || t_end > groups) throw SimError("loop range outside [0, 2^(n-k))");
    use_device(st->ctx);
    GateMatrix over;
    if (matrix_override) {
      over = GateMatrix(kp.gate.k());
      for (size_t i = 0; i < over.entries().size(); ++i)
        over.entries()[i] = cplx(matrix_override[2 * i], matrix_override[2 * i + 1]);
    }
    const LaunchStructure ls = derive_launch(kp, matrix_override ? &over : nullptr, st->prec);
    tsg::GateLaunch g = make_launch(kp, ls);
    g.re = st->re;
    g.im = st->im;
    g.g_begin = t_begin;
    g.g_end = t_end;
    g.full_range = t_begin == 0 && t_end == groups;
    choose_dmma_perm(g, ls);
    if (t_begin == t_end) return TSG_OK;
    if (needs_tile_matrix(g, st->prec)) {
      const auto bytes = tile_matrix_bytes(ls, g);
      if (p->dev_mat_bytes < bytes.size()) {
        if (p->dev_mat) ck(cudaFree(p->dev_mat), "cudaFree");
        ck(cudaMalloc(&p->dev_mat, bytes.size()), "cudaMalloc plan matrix");
        p->dev_mat_bytes = bytes.size();
      }
      ck(cudaMemcpyAsync(p->dev_mat, bytes.data(), bytes.size(), cudaMemcpyHostToDevice, st->stream), "matrix upload");
      g.dev_mat = p->dev_mat;
    }
    launch(st, g);
  })
}

// --------------------------------------------------------------- programs
int tsg_program_create(tsg_ctx* ctx, const tsc_circuit* fused, double zero_tol, double one_tol, int precision_bits,
                       tsg_program** out) {
  TSG_TRY({
    require(ctx && fused && out, "null argument");
    require(precision_bits == 64 || precision_bits == 32, "precision_bits must be 64 or 32");
    *out = build_program(ctx, fused->c, zero_tol, one_tol, precision_bits).release();
  })
}

int tsg_program_destroy(tsg_program* prog) {
  if (!prog) return TSG_OK;
  cudaSetDevice(prog->ctx->device);
  for (auto& kv : prog->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
  }
  if (prog->arena) cudaFree(prog->arena);
  if (prog->ev0) cudaEventDestroy(prog->ev0);
  if (prog->ev1) cudaEventDestroy(prog->ev1);
  delete prog;
  return TSG_OK;
}

static void fill_report(const tsg_program* prog, double exec_s, tsg_run_report* r) {
  if (!r) return;
  r->planning_s = prog->planning_s;
  r->execution_s = exec_s;
  r->gates = prog->gates.size();
  r->launches = prog->launches;
  r->bytes = prog->bytes;
  r->touched_bytes = prog->touched_bytes;
  r->total_op_count = prog->total_ops;
  r->exchanged_bytes = 0;
  r->exchange_s = 0.0;
}

static cudaGraphExec_t program_graph(tsg_state* st, tsg_program* prog) {
  auto key = std::make_pair(st, st->serial);
  auto it = prog->graphs.find(key);
  if (it == prog->graphs.end()) {
    // relaxed capture: first-use kernel attributes may be set while capturing
    tsg_program::Graph gr;
    ck(cudaStreamBeginCapture(st->stream, cudaStreamCaptureModeRelaxed), "begin capture");
    try {
      run_program(st, prog, nullptr);
    } catch (...) {
      cudaGraph_t dummy = nullptr;
      cudaStreamEndCapture(st->stream, &dummy);
      if (dummy) cudaGraphDestroy(dummy);
      throw;
    }
    ck(cudaStreamEndCapture(st->stream, &gr.graph), "end capture");
    ck(cudaGraphInstantiate(&gr.exec, gr.graph, 0), "graph instantiate");
    it = prog->graphs.emplace(key, gr).first;
  }
  return it->second.exec;
}

// Graphs pay off on reuse: the first run of a program on a state launches
// its kernels directly (no capture / instantiate on a one-shot run), later
// runs replay a captured graph.
static bool graph_ready(tsg_state* st, tsg_program* prog, int use_graph) {
  if (!use_graph) return false;
  const auto key = std::make_pair(st, st->serial);
  if (prog->graphs.count(key)) return true;
  return ++prog->uses[key] > 1;
}

static void enqueue_program(tsg_state* st, tsg_program* prog, int use_graph) {
  require(st->n == prog->n && st->prec == prog->prec, "program was built for a different state shape");
  use_device(st->ctx);
  if (use_graph) ck(cudaGraphLaunch(program_graph(st, prog), st->stream), "graph launch");
  else run_program(st, prog, nullptr);
}

int tsg_program_enqueue(tsg_state* st, tsg_program* prog, int use_graph) {
  TSG_TRY({
    require(st && prog, "null argument");
    enqueue_program(st, prog, graph_ready(st, prog, use_graph));
  })
}

int tsg_program_run(tsg_state* st, tsg_program* prog, int use_graph, tsg_run_report* report) {
  TSG_TRY({
    require(st && prog, "null argument");
    const bool graph = graph_ready(st, prog, use_graph);
    if (graph) program_graph(st, prog);  // capture before the timed events
    ck(cudaEventRecord(prog->ev0, st->stream), "event");
    enqueue_program(st, prog, graph);
    ck(cudaEventRecord(prog->ev1, st->stream), "event");
    ck(cudaEventSynchronize(prog->ev1), "run sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, prog->ev0, prog->ev1), "elapsed");
    fill_report(prog, ms * 1e-3, report);
  })
}

int tsg_program_run_profiled(tsg_state* st, tsg_program* prog, double* seconds, tsg_run_report* report) {
  TSG_TRY({
    require(st && prog, "null argument");
    require(st->n == prog->n && st->prec == prog->prec, "program was built for a different state shape");
    use_device(st->ctx);
    std::vector<cudaEvent_t> marks(prog->gates.size() + 1);
    for (auto& e : marks) ck(cudaEventCreate(&e), "event");
    run_program(st, prog, &marks);
    ck(cudaEventSynchronize(marks.back()), "run sync");
    double total = 0.0;
    for (size_t i = 0; i < prog->gates.size(); ++i) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, marks[i], marks[i + 1]), "elapsed");
      if (seconds) seconds[i] = ms * 1e-3;
      total += ms * 1e-3;
    }
    for (auto& e : marks) cudaEventDestroy(e);
    fill_report(prog, total, report);
  })
}

int tsg_program_gate_info(const tsg_program* prog, uint64_t i, tsg_plan_info* out) {
  TSG_TRY({
    require(prog && out, "null argument");
    require(i < prog->gates.size(), "gate index out of range");
    fill_info(prog->gates[i].plan, prog->gates[i].ls, out);
    out->batched = prog->gates[i].in_batch ? 2 : (prog->gates[i].batch >= 0 ? 1 : 0);
    if (out->batched == 1) out->touched_fraction = 1.0;
    if (out->batched == 2) out->touched_fraction = 0.0;
  })
}

int tsg_program_step_count(const tsg_program* prog, uint64_t* out) {
  TSG_TRY({
    require(prog && out, "null argument");
    *out = prog->steps.size();
  })
}

int tsg_program_jit_kernels(const tsg_program* prog, int* jit_passes, int* jit_gate_launches) {
  TSG_TRY({
    require(prog && jit_passes && jit_gate_launches, "null argument");
    *jit_passes = *jit_gate_launches = 0;
    for (const ProgramPass& pp : prog->passes) *jit_passes += pp.launch.jit != nullptr;
    for (const ProgramStep& st : prog->steps) {
      if (st.kind != kStepGate) continue;
      const ProgramGate& pg = prog->gates[st.gate];
      if (pg.subs.empty()) *jit_gate_launches += pg.launch.jit != nullptr;
      for (const tsg::GateLaunch& g : pg.subs) *jit_gate_launches += g.jit != nullptr;
    }
  });
}

int tsg_program_pass_layouts(const tsg_program* prog, uint64_t i, int* smem_layouts, int* shuffle_layouts) {
  TSG_TRY({
    require(prog && smem_layouts && shuffle_layouts, "null argument");
    require(i < prog->steps.size(), "step index out of range");
    const ProgramStep& st = prog->steps[i];
    *smem_layouts = *shuffle_layouts = 0;
    if (st.kind == kStepPass) {
      *smem_layouts = prog->passes[st.index].layouts_smem;
      *shuffle_layouts = prog->passes[st.index].layouts_shuffle;
    }
  });
}

int tsg_program_step_info(const tsg_program* prog, uint64_t i, tsg_step_info* out) {
  TSG_TRY({
    require(prog && out, "null argument");
    require(i < prog->steps.size(), "step index out of range");
    const ProgramStep& st = prog->steps[i];
    std::memset(out, 0, sizeof *out);
    out->kind = st.kind;
    out->first_gate = static_cast<uint64_t>(st.gate);
    out->n_gates = static_cast<uint64_t>(st.n_gates);
    std::string name;
    if (st.kind == kStepPermute) {
      const size_t sweeps = prog->permutes[st.index].invs.size();
      name = sweeps == 1 ? "k_permute" : "k_permute x" + std::to_string(sweeps);
    } else if (st.kind == kStepPass) {
      const ProgramPass& pp = prog->passes[st.index];
      out->n_high = pp.launch.tile_log2 - pp.launch.run_log2;
      for (int h = 0; h < out->n_high; ++h) out->high[h] = pp.launch.high[h];
      name = pp.launch.jit ? "k_pass_jit" : "k_pass";
    } else if (st.kind == kStepBatch) {
      name = "k_diag_batch";
    } else if (!prog->gates[st.gate].subs.empty()) {  // block split: "<part kernel> xN split"
      const ProgramGate& pg = prog->gates[st.gate];
      tsg::GateLaunch g = pg.subs[0];
      if (pg.sub_mat[0] != SIZE_MAX) g.dev_mat = prog->arena;
      name = tsg::kernel_name(g, prog->prec) + " x" + std::to_string(pg.subs.size()) + " split";
    } else {
      tsg::GateLaunch g = prog->gates[st.gate].launch;
      if (prog->gates[st.gate].has_mat) g.dev_mat = prog->arena;
      name = tsg::kernel_name(g, prog->prec);
    }
    std::strncpy(out->kernel, name.c_str(), sizeof(out->kernel) - 1);
  })
}

// bench_cost_model on the device.  For k in [1, k_max] and
// density levels {diagonal, quarter, half, dense} (the diagonal level is a
// B200 addition: diagonal gates run on the streaming kernel and are the
// cheapest class), a seeded random gate on two random target sets is planned
// exactly as run_circuit plans it and timed with CUDA events on a 2^bench_n
// scratch state; spg = median seconds / 2^(n-k).  `threads` is recorded as 1
// (one device); the host string names the device and clocks.
int tsg_bench_cost_model(tsg_ctx* ctx, int bench_n, int k_max, int precision_bits, int repetitions, uint64_t seed,
                         tsc_cost_model** out) {
  if (!ctx) {
    tsg_detail::set_error("null argument");
    return TSG_ERR_CONFIG;
  }
  const int full = ctx->num_sms;
  return tsg_bench_cost_model_sms(ctx, bench_n, k_max, precision_bits, repetitions, seed, &full, 1, out);
}

// The B200 form of SPEC's `threads` axis (kernels timed per
// worker count): the number of SMs the persistent grids of the gate kernels
// span.  Every (k, density) point is timed once per SM count; records carry
// threads = that SM count (the full device: ctx's SM count).
int tsg_bench_cost_model_sms(tsg_ctx* ctx, int bench_n, int k_max, int precision_bits, int repetitions, uint64_t seed,
                             const int* sm_counts, int n_sm_counts, tsc_cost_model** out) {
  TSG_TRY({
    require(ctx && out && sm_counts && n_sm_counts >= 1, "null argument");
    for (int i = 0; i < n_sm_counts; ++i)
      require(sm_counts[i] >= 1 && sm_counts[i] <= ctx->num_sms, "SM counts must be in [1, the device's SM count]");
    require(bench_n >= 8 && bench_n <= 34, "bench_n must be in [8, 34]");
    require(k_max >= 1 && k_max <= 6 && k_max < bench_n, "k_max must be in [1, 6]");
    require(repetitions >= 1, "repetitions must be >= 1");
    tsg_state* st = nullptr;
    if (int rc = tsg_state_create(ctx, bench_n, precision_bits, &st)) throw SimError(tsg_last_error());
    std::unique_ptr<tsg_state, int (*)(tsg_state*)> guard(st, tsg_state_destroy);
    if (int rc = tsg_state_init_random(st, seed)) throw SimError(tsg_last_error());
    CostModel cm;
    cm.bench_n = bench_n;
    cm.precision = precision_bits == 64 ? "f64" : "f32";
    cm.host = ctx->name + " sm_100a, " + std::to_string(ctx->num_sms) + " SMs, CUDA-event timed";
    Prng rng(seed);
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    void* dev_mat = nullptr;
    ck(cudaMalloc(&dev_mat, 3 * 4096 * sizeof(double)), "cudaMalloc bench matrix");
    for (int k = 1; k <= k_max; ++k) {
      for (int level = 0; level < 4; ++level) {  // 0 diag, 1 quarter, 2 half, 3 dense
        std::vector<std::vector<double>> times(n_sm_counts);
        uint64_t ops = 0;
        for (int trial = 0; trial < 2; ++trial) {
          std::vector<int> pool(bench_n);
          for (int i = 0; i < bench_n; ++i) pool[i] = i;
          for (int i = bench_n - 1; i > 0; --i) std::swap(pool[i], pool[rng.next_below(i + 1)]);
          std::vector<int> targets(pool.begin(), pool.begin() + k);
          std::sort(targets.begin(), targets.end());
          GateMatrix m = random_unitary(k, rng);
          const uint64_t D = m.dim();
          if (level == 0) {
            for (uint64_t r = 0; r < D; ++r)
              for (uint64_t c = 0; c < D; ++c)
                if (r != c) m.at(r, c) = 0.0;
          } else if (level < 3) {
            const double keep = level == 1 ? 0.25 : 0.5;
            for (uint64_t r = 0; r < D; ++r)
              for (uint64_t c = 0; c < D; ++c)
                if (r != c && rng.uniform() >= keep) m.at(r, c) = 0.0;
          }
          KernelPlan plan = plan_kernel(make_gate(m, targets), bench_n, 0, 1e-8, 1e-8, false);
          const LaunchStructure ls = derive_launch(plan, nullptr, precision_bits);
          tsg::GateLaunch g = make_launch(plan, ls);
          g.re = st->re;
          g.im = st->im;
          if (needs_tile_matrix(g, precision_bits)) {
            const auto bytes = tile_matrix_bytes(ls, g);
            ck(cudaMemcpy(dev_mat, bytes.data(), bytes.size(), cudaMemcpyHostToDevice), "bench matrix upload");
            g.dev_mat = dev_mat;
          }
          ops = std::max(ops, plan.profile.op_count);
          for (int t = 0; t < n_sm_counts; ++t) {
            // the same state and stream, launches sized for sm_counts[t] SMs
            tsg_ctx sub = *ctx;
            sub.num_sms = sm_counts[t];
            tsg_state view = *st;
            view.ctx = &sub;
            launch(&view, g);  // warm-up (first-use kernel attributes)
            for (int r = 0; r < repetitions; ++r) {
              ck(cudaEventRecord(e0, st->stream), "event");
              launch(&view, g);
              ck(cudaEventRecord(e1, st->stream), "event");
              ck(cudaEventSynchronize(e1), "event sync");
              float ms = 0.f;
              ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
              times[t].push_back(ms * 1e-3);
            }
          }
        }
        for (int t = 0; t < n_sm_counts; ++t) {
          std::sort(times[t].begin(), times[t].end());
          const double med = times[t][times[t].size() / 2];
          CostRecord rec;
          rec.k = k;
          rec.op_count = ops;
          rec.threads = sm_counts[t];
          rec.seconds_per_group = std::max(med, 1e-9) / std::ldexp(1.0, bench_n - k);
          cm.records.push_back(rec);
        }
      }
    }
    cudaFree(dev_mat);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = new tsc_cost_model{std::move(cm)};
  })
}

}  // extern "C"

#include "shard_exec.cuh"
