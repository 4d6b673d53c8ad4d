// tilesim/pass.hpp -- grouping of a fused gate stream into tile passes.
//
// B200 addition to run_circuit.  The reference applies
// every fused gate with its own sweep over the state (one apply_kernel call
// per gate, a barrier between gates); on B200 each sweep is
// a full HBM read + write of the state (2 * 2^n * B_amp bytes).  A *pass*
// applies a run of consecutive gates in one sweep: the state is cut into
// tiles of 2^M amplitudes spanned by the low run qubits [0, L) and M - L
// "high" tile qubits; a gate can join the pass when every qubit it mixes is
// a tile qubit (controls and diagonal targets may sit anywhere -- their value
// is a constant of the tile).  Gates keep their program order and their
// per-gate arithmetic; only the number of HBM sweeps changes.
#pragma once

#include <cstdint>
#include <vector>

#include "tilesim/plan.hpp"

namespace tilesim {

struct PassConfig {
  int tile_log2 = 11;    // M: amplitudes per tile = 2^M
  int run_log2 = 5;      // L: contiguous run length = 2^L (>= 256 bytes per array)
  int max_ops = 96;      // ops per pass
  int max_gen_ks = 4;    // widest non-diagonal sub-gate inside a pass
  int max_blob = 32 * 1024;  // bytes of run offsets + op table + op data
  int amp_real_bytes = 8;    // sizeof(Real) of the state
  // B200 cost model of a pass, in units of one state sweep (2 * 2^n * B_amp
  // bytes at HBM speed), measured with scripts/pass_bench.py at n = 28
  // (profiles/r01/pass_bench.txt): the pass itself, each diagonal op, each
  // GEN op by mixed-qubit count (register ops up to reg_bits mixed qubits,
  // shared-memory ops above; layout changes included), monomial ops; a
  // standalone launch costs its sweep (touched share for controlled gates).
  double base_sweeps = 1.07;
  double diag_sweeps = 0.04;
  double gen_sweeps[6] = {0.0, 0.2, 0.45, 0.6, 1.2, 2.0};
  double perm_sweeps_reg = 0.4;
  double perm_sweeps_smem = 0.5;
  double standalone_sweeps = 1.08;
  int reg_bits = 3;  // register positions a register op may mix (2^M / 256 amplitudes per thread)
  // a run of at least this many consecutive qubit-permutation gates (SWAP
  // layers) becomes one permutation step: one in-place sweep (two for a
  // permutation that is not an involution) instead of a sweep per gate
  int min_permute_run = 3;
  // testing: every eligible gate joins (no cost test, single-gate passes allowed);
  // pass_config() sets it when the environment has TSG_PASS_FORCE=1
  bool force = false;
};

// Whether a program over n qubits gets JIT-compiled passes (the runtime's
// rule: TSG_PASS_JIT=0 disables, TSG_PASS_JIT_MIN_N, default 24).
bool pass_jit_expected(int n_qubits);
// Defaults per state precision (64: complex128, 32: complex64); the op costs
// are those of the kernel the passes of an n-qubit program will run (the JIT
// pass or the interpreter; n_qubits = 0: the interpreter's).
PassConfig pass_config(int precision_bits, int n_qubits = 0);

enum class PassRole : int { Standalone = 0, Diag = 1, Gen = 2 };

// The sub-targets a non-diagonal sub-gate actually mixes: bit b of the
// sub-gate is a *block* bit when every nonzero entry M[r][c] has
// r_b == c_b (the matrix is block-diagonal in that qubit, e.g. the phase
// qubits of a fused QFT block); the remaining bits are *mixed*.  Only mixed
// qubits must be tile qubits -- block bits select one of 2^|B| blocks and,
// like controls, may sit anywhere.  Returns positions (0..ks-1) of the mixed
// bits, ascending.
std::vector<int> mixed_bits(const LaunchStructure& ls);

// Every row of the snapped sub-matrix has exactly one nonzero entry (a
// permutation with phases): a pass applies it as a gather (Perm op).
bool monomial(const LaunchStructure& ls);

// Block decomposition of a non-diagonal sub-gate over its block bits: one
// launch structure per block value, with the block qubits added to the
// controls (the plan's exact-identity control peeling, generalised to
// non-identity blocks).  Identity blocks are dropped.  Every result touches
// 2^-|B| of the state with a 2^|E|-qubit sub-gate, so a 5-qubit gate with one
// block qubit costs two 4-qubit half-sweeps instead of one FP64-bound
// 5-qubit sweep.  Returns {ls} when every bit is mixed.
std::vector<LaunchStructure> split_blocks(const LaunchStructure& ls, int precision_bits);

// A sub-gate without controls whose snapped matrix is a 0/1 permutation that
// moves bit b of the sub-index to bit sigma[b] (SWAP and products of SWAPs,
// e.g. QFT's bit-reversal layer after fusion): the gate permutes qubits.
bool qubit_permutation(const LaunchStructure& ls, std::vector<int>* sigma);

// How one gate can be executed inside a pass (or not at all).
PassRole pass_role(const LaunchStructure& ls, const PassConfig& cfg);

// Bytes the op occupies in the pass blob (PassOp record + its data).
int pass_op_bytes(const LaunchStructure& ls, const PassConfig& cfg);

struct PassStep {
  bool is_pass = false;
  bool is_permute = false;  // a run of qubit-permutation gates (qubit_permutation), one k_permute step
  std::vector<int> gates;  // program gate indices, program order
  std::vector<int> high;   // pass only: the M - L high tile qubits, ascending
};

// Estimated cost (sweeps) of a gate inside a pass / launched on its own.
double pass_op_sweeps(const LaunchStructure& ls, const PassConfig& cfg);
double standalone_sweeps(const LaunchStructure& ls, const PassConfig& cfg);

// Greedy in program order: extend the current pass while the gate is cheaper
// inside it than on its own, the union of the mixed qubits above L fits
// M - L and the blob / op budgets hold; a finished pass whose estimated cost
// exceeds that of launching its gates one by one is emitted as standalone
// gates.  Identity gates (nothing to launch) are dropped.  Runs of at least
// min_permute_run consecutive qubit-permutation gates become one permutation
// step (is_permute).
std::vector<PassStep> plan_passes(const std::vector<LaunchStructure>& gates, int n, const PassConfig& cfg);

}  // namespace tilesim
