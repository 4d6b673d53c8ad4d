// Host/device-neutral description of one gate launch, built on the host from
// a KernelPlan's LaunchStructure (include/tilesim/plan.hpp) and consumed by
// the per-precision launchers in apply_f64.cu / apply_f32.cu.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace tsg {

constexpr int kMaxMasks = 13;  // k + 1 startIdx masks, k <= 12
constexpr int kMaxSub = 6;     // largest non-diagonal sub-gate on the GPU

struct GateLaunch {
  int klass = 0;   // tilesim::KernelClass
  int k = 0;       // gate size (all targets, controls included)
  int ks = 0;      // sub-gate size
  int sparse = 0;  // zero-skipping variant
  int n = 0;       // qubits of the state
  void* re = nullptr;
  void* im = nullptr;
  // group range [g_begin, g_end) of the s = 0 loop counter over 2^(n-k)
  uint64_t g_begin = 0, g_end = 0;
  bool full_range = true;
  uint64_t masks[kMaxMasks] = {};
  int n_masks = 0;
  uint64_t fixed_or = 0;            // active control values
  int n_ctrl = 0;
  int ctrl[12] = {};                // control qubits, ascending
  int sub_targets[12] = {};         // sub-gate qubits, ascending
  uint64_t off[1 << kMaxSub] = {};  // deposit of j over sub_targets
  const double* m_re = nullptr;     // host: snapped sub-matrix, row-major
  const double* m_im = nullptr;
  const void* dev_mat = nullptr;    // device copy for Tile: [D*D re][D*D im] in state precision
};

// Launch on `stream`; returns the number of kernels enqueued (0 for identity).
int launch_gate_f64(const GateLaunch& g, cudaStream_t stream, int num_sms);
int launch_gate_f32(const GateLaunch& g, cudaStream_t stream, int num_sms);

// A run of consecutive full-range diagonal gates applied in ONE streaming
// pass.  Per element the gates are applied in program order with exactly the
// arithmetic of k_diag, so the result is bit-identical to separate launches.
constexpr int kMaxBatch = 16;
constexpr int kMaxBatchEntries = 1024;  // sum of 2^ks over the batch
struct DiagBatchLaunch {
  int n = 0;  // qubits
  void* re = nullptr;
  void* im = nullptr;
  int n_gates = 0;
  uint64_t cmask[kMaxBatch] = {};  // control qubits of gate g
  uint64_t cval[kMaxBatch] = {};   // their active values
  int ks[kMaxBatch] = {};
  int tq[kMaxBatch][6] = {};       // sub-target qubits
  int toff[kMaxBatch] = {};        // table offset of gate g
  int n_entries = 0;
  const double* tables = nullptr;  // device: interleaved (re, im) diagonal entries, FP64
};
int launch_diag_batch_f64(const DiagBatchLaunch& b, cudaStream_t stream, int num_sms);
int launch_diag_batch_f32(const DiagBatchLaunch& b, cudaStream_t stream, int num_sms);

// Name of the kernel template a launch selects (for reports / profiles).
const char* kernel_name(const GateLaunch& g, int precision_bits);

}  // namespace tsg
