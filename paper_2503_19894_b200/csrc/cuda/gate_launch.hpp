// Host/device-neutral description of one gate launch, built on the host from
// a KernelPlan's LaunchStructure (include/tilesim/plan.hpp) and consumed by
// the per-precision launchers in apply_f64.cu / apply_f32.cu.
#pragma once

#ifndef __CUDACC_RTC__  // NVRTC (pass_jit.cpp) supplies the integer types
#include <cstdint>
#include <string>

#include <cuda_runtime.h>
#endif

namespace tsg {

// constexpr bit helpers usable in templates on both compilers
__host__ __device__ constexpr int cx_popc(unsigned x) { return x ? int(x & 1u) + cx_popc(x >> 1) : 0; }
__host__ __device__ constexpr int cx_ctz(unsigned x) { return (x & 1u) || !x ? 0 : 1 + cx_ctz(x >> 1); }

constexpr int kMaxMasks = 13;  // k + 1 startIdx masks, k <= 12
constexpr int kMaxSub = 6;     // largest non-diagonal sub-gate on the GPU

// Insertion masks (SPEC.md:441-449 form) for zeros at sorted `pos` inside a
// value of `width` bits: x -> sum_i (x & m[i]) << i.
inline int insertion_masks(const int* pos, int count, int width, uint64_t* out) {
  int from = 0;
  for (int i = 0; i <= count; ++i) {
    const int to = i < count ? pos[i] - i : width;
    uint64_t m = 0;
    for (int b = from; b < to && b < width; ++b) m |= uint64_t{1} << b;
    out[i] = m;
    from = to > from ? to : from;
  }
  return count + 1;
}

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
  // Element order of the DMMA kernels: row / column j of dev_mat is row /
  // column perm[j] of the sub-gate (a qubit reordering chosen on the host so
  // that zero structure falls into whole 8x4 DMMA tiles).  Identity unless
  // the full-range DMMA path runs.
  uint8_t perm[1 << kMaxSub] = {};
  // complex128 DMMA product JIT-compiled with this launch's zero 8 x 4 tiles
  // compiled in (dmma_jit_spec, pass_jit.hpp); null: the generic kernel
  const void* jit = nullptr;
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

#ifndef __CUDACC_RTC__
// Name of the kernel template a launch selects (for reports / profiles).
std::string kernel_name(const GateLaunch& g, int precision_bits);
#endif

// ------------------------------------------------------------ tile passes
// A pass applies a run of fused gates to the state in ONE read + write of
// HBM (k_pass, kernels_pass.cuh).  The state is cut into tiles of 2^M
// amplitudes: the "tile qubits" are the low run bits [0, L) plus M - L high
// qubits; every other qubit is fixed per tile.  A gate joins a pass when its
// non-control sub-targets are tile qubits (GEN op) or when it is diagonal
// (DIAG op: out-of-tile targets and controls are constants of the tile).
// Tile coordinates: position p < L is qubit p; position L + h is high[h].
constexpr int kPassThreads = 256;  // threads per CTA, two CTAs per SM
constexpr int kPassLogThreads = 8;
constexpr int kPassMaxOps = 128;  // ops + RUN headers per pass
constexpr int kPassMaxBlob = 32 * 1024;  // run offsets + op table + op data, staged in smem
constexpr int kPassMaxGEntries = 128;    // combined diagonal-group entries per run (smem scratch)
constexpr int kPassMaxSig = 6;           // signature bits of a diagonal group
constexpr int kPassPadBytes = 32;        // padding between runs in shared memory (bank spread)

// Register layouts.  Each consumer thread holds R = 2^r = 2^M / kPassThreads
// amplitudes of the tile in registers: a LAYOUT op picks r "register" tile
// positions P; thread tid holds x = deposit(tid over the other positions) |
// deposit(i over P), i < R.  Ops run on those registers; only a layout
// change or a wide op moves the tile through shared memory.
//   Layout  store the registers (old layout), barrier, load the new layout
//   Run     header of a run of diagonal ops (diagonal gates commute).  Ops
//           are grouped by signature -- the in-tile positions their targets
//           and controls touch (at most 6): per tile, the CTA builds each
//           group's combined table over its signature once (out-of-tile
//           bits and controls are tile constants), then every amplitude
//           takes one lookup per group.  Ops with wider signatures follow
//           as per-op classes w.r.t. the current layout:
//     DiagT  in-tile index bits only on thread positions: one factor per thread
//     DiagI  only on register positions: one factor per register index i,
//            shared through shared memory
//     DiagX  both: a table lookup per amplitude
//   RGen    sub-gate whose mixed qubits are register positions (rmask): in
//           registers, one block (tilesim::mixed_bits) per sub-group
//   RPerm   RGen whose blocks are monomial (one nonzero per row: X, CX, SWAP,
//           permutations with phases): a select and one complex multiply
//   SGen / SPerm  mixed qubits not all register positions (or more than r):
//           through shared memory, one thread (or a row split) per group
enum PassOpKind : int32_t {
  kPassLayout = 0,
  kPassRun = 1,
  kPassDiagT = 2,
  kPassDiagI = 3,
  kPassDiagX = 4,
  kPassRGen = 5,
  kPassRPerm = 6,
  kPassSGen = 7,
  kPassSPerm = 8,
  kPassDGroup = 9,   // RUN group header: diagonal ops sharing an in-tile signature
  kPassDMember = 10, // member of the preceding DGroup
};

struct PassOp {  // 192 bytes, built on the host, read from shared memory
  int32_t kind;
  int32_t ks;           // DIAG: table bits; GEN / PERM: mixed qubits; RUN: number of DiagT ops
  int32_t data_off;     // byte offset of the op's data in the blob
  int32_t n_out;        // table / block index bits taken from the tile base (out_gbit -> out_jbit)
  int32_t log2_groups;  // SGen / SPerm: groups per tile; RUN: number of DiagI ops
  int32_t log2_rsplit;  // SGen / SPerm: rows of a group split over 2^log2_rsplit threads; RUN: number of DiagX ops
  int32_t aux_off;      // DiagT / DiagX: thread table; GEN / PERM: blocks
  int32_t rmask;        // RGen / RPerm: mixed bits among the register bits
  uint32_t ictl_mask, ictl_val;  // controls on register bits (DIAG, RGen, RPerm)
  uint32_t tctl_mask, tctl_val;  // RGen / RPerm: controls on thread positions (tile coordinates)
  uint64_t cout_mask, cout_val;  // controls outside the tile (global bits)
  uint8_t out_gbit[8], out_jbit[8];
  uint32_t dep[8];    // DIAG: table bits per register bit; RGen / RPerm: block bits per register bit;
                      // LAYOUT: padded shared-memory offset of register position k
  uint32_t xmask[6];  // LAYOUT: insertion masks, thread id -> thread positions (zeros at P; r + 1 <= 6)
  uint8_t tb_pos[8], tb_jbit[8];  // RGen / RPerm: block bits on thread positions
  int32_t n_tb;
  int32_t n_xmask;
  int32_t thr_off;  // RGen / RPerm: per-thread u8 table (block bits from thread positions, 0xff: thread
                    // controls inactive), -1 when the op has neither
  // LAYOUT in registers (warp shuffles): the new layout swaps register bit
  // swap_k[s] with lane bit swap_l[s], s < n_swap (0: through shared memory)
  int32_t n_swap;
  uint8_t swap_k[4], swap_l[4];
  uint8_t reserved[16];
};
static_assert(sizeof(PassOp) == 192, "PassOp layout");

// Blob: [run offsets: 2^(M-L) x u64][PassOp x n_ops][op data].  Op data:
//   DIAG   table[2^ks + 1] {re, im} (state precision; the last entry is 1 and
//          stands in for inactive controls); DiagT / DiagX also thr[256] u8
//          at aux_off: table-index bits on thread positions, 0xff when the
//          controls on thread positions are inactive for that thread
//   RGen   at aux_off the 2^nb blocks, 2^ks x 2^ks {re, im} row-major, one
//          padding entry after each block (stride 4^ks + 1)
//   RPerm  at aux_off per block: src[2^ks] u32 (element index of the source
//          of row r; 16-byte block) and val[2^ks] {re, im}
//   SGen   soff[2^ks] u32 (16-byte block), et[256] u32, ek[max(1, groups/256)] u32:
//          group g = tid + 256 k sits at padded offset (et[tid] + ek[k]) & 0xffff
//          and uses block ((et[tid] + ek[k]) >> 16) | (bits from the tile base);
//          then the blocks as for RGen
//   SPerm  as SGen up to aux_off; there, per block: src[2^ks] u32 (padded
//          offset of the source element of each row; 16-byte block) and
//          val[2^ks] {re, im}
struct PassLaunch {
  int n = 0;          // state qubits
  int tile_log2 = 0;  // M
  int run_log2 = 0;   // L
  int high[16] = {};  // tile qubits >= L, ascending (M - L of them)
  void* re = nullptr;
  void* im = nullptr;
  const void* blob = nullptr;  // device
  int blob_bytes = 0;
  int n_ops = 0;
  const void* jit = nullptr;   // JIT-compiled kernel of this op table (pass_jit.cu), else the interpreter
};
int launch_pass_f64(const PassLaunch& p, cudaStream_t stream, int num_sms);
int launch_pass_f32(const PassLaunch& p, cudaStream_t stream, int num_sms);

// ---------------------------------------------------------- permutations
// A run of qubit-permutation gates (SWAP layers) applied as ONE involutive
// qubit permutation of the state, in place: new[y] = old[P(y)] with P moving
// index bit q to p[q], p an involution (permute.cu).
struct PermuteLaunch {
  int n = 0;
  void* re = nullptr;
  void* im = nullptr;
  int p[64] = {};
};
int launch_permute_f64(const PermuteLaunch& p, cudaStream_t stream, int num_sms);
int launch_permute_f32(const PermuteLaunch& p, cudaStream_t stream, int num_sms);

}  // namespace tsg
