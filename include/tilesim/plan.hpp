// tilesim/plan.hpp -- kernel plans.
//
//   QubitSplit / split_qubits     SPEC.md:412-417, 432-440 (Fig. 6 colouring)
//   MaskTable / build_masks       SPEC.md:418-423, 441-449 (startIdx masks)
//   KernelPlan / plan_kernel
//
// B200 additions (host side, no CUDA): every plan also carries the launch
// structure the sm_100a kernels consume -- the matrix snapped to its scalar
// kinds, the control qubits peeled off (rows/cols that are exact identity),
// the remaining sub-gate, and the kernel class that applies it.  The GPU
// kernels run in the s = 0 group space of the paper's GPU ABI:
// group t in [0, 2^(n-k)), base = startIdx(t) over all k targets.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tilesim/core.hpp"

namespace tilesim {

struct QubitSplit {
  int s = 0;
  std::vector<int> lower;   // Q ∩ L
  std::vector<int> higher;  // Q ∩ H
  std::vector<int> red;     // the s smallest non-target indices
  int k_L = 0, k_H = 0, lower_region_size = 0;
};

struct MaskTable {
  std::vector<uint64_t> masks;  // k_H + 1 disjoint masks over t
};

struct EntryOp {
  uint32_t row, col;
  ScalarKind re_kind, im_kind;
  double re, im;
};

// How a plan is executed on the GPU.
enum class KernelClass : int {
  Identity = 0,  // the snapped sub-gate is the identity: nothing to launch
  Diagonal = 1,  // streaming multiply by a diagonal over the active slice
  Direct = 2,    // one thread per group, amplitudes and matrix in registers
  Tile = 3,      // CTA-cooperative smem tile: the group batch times the matrix
};
const char* to_string(KernelClass k);

struct LaunchStructure {
  KernelClass klass = KernelClass::Direct;
  std::vector<int> controls;     // qubits whose inactive half is untouched
  uint64_t control_values = 0;   // active value of each control at its qubit bit
  std::vector<int> sub_targets;  // remaining qubits, ascending
  int ks = 0;                    // |sub_targets|
  std::vector<uint64_t> offsets; // 2^ks: deposit of j over sub_targets
  std::vector<double> sub_re, sub_im;  // snapped 2^ks x 2^ks sub-matrix
  uint64_t nonzero_scalars = 0;  // in the sub-matrix
  bool sparse = false;           // prefer the zero-skipping variant
};

struct KernelPlan {
  Gate gate;
  int n = 0;
  QubitSplit split;
  MaskTable mask_table;      // for the plan's s
  MaskTable group_masks;     // s = 0 masks, used by the GPU kernels
  std::vector<EntryOp> entry_ops;  // entries whose two scalars are not both Zero
  SparsityProfile profile;
  double zero_tol = 1e-8, one_tol = 1e-8;
  bool runtime_matrix = false;
  LaunchStructure launch;
  uint64_t loop_count() const { return uint64_t{1} << (n - gate.k() - split.s); }
};

QubitSplit split_qubits(const std::vector<int>& targets, int s);
MaskTable build_masks(const QubitSplit& split, int n);
uint64_t start_index(uint64_t t, const MaskTable& m);

// Throws ConfigError when k + s > n (k + s == n is a 1-iteration loop and is
// accepted; SPEC.md:454 rejects it -- documented deviation).
KernelPlan plan_kernel(const Gate& g, int n, int s, double zero_tol, double one_tol, bool runtime_matrix);

// Launch structure for a (possibly overridden) matrix with the plan's kinds.
// Throws SimError when an override scalar does not classify to the planned
// kind.
LaunchStructure derive_launch(const KernelPlan& plan, const GateMatrix* override_matrix, int precision_bits);

std::string describe(const KernelPlan& p);  // SPEC.md:493 plan dump

}  // namespace tilesim
