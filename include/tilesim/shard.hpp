// tilesim/shard.hpp -- global-qubit sharding of the statevector (new layer;
// the reference's SPEC lists distributed statevectors as a non-goal,
// SPEC.md:567, so this is the B200 extension of north-star item 3).
//
// 2^g ranks each hold 2^(n-g) amplitudes.  Physical index bits [0, n_local)
// address a rank's local array; bits [n_local, n) are the rank id.  A
// logical->physical qubit map evolves as qubits are swapped:
//
//   Local      every target is local: apply on each rank (physical targets)
//   RankBlock  the gate is block-diagonal in its global target bits (CP, CZ,
//              RZ, fused ZZ phases, a controlled-U with a global control):
//              rank r applies the sub-block selected by its own bits -- no
//              communication (SURVEY.md §8e "exchange-free cases")
//   Swap       exchange a global position with a local one: ranks r and
//              r ^ 2^i swap the halves whose local bit differs from rank bit i
//              (2^(n_local-1) amplitudes each way); the highest free local
//              positions are chosen so the exchanged halves are contiguous
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "tilesim/ir.hpp"

namespace tilesim {

struct ShardOp {
  enum class Kind { Local, RankBlock, Swap };
  Kind kind = Kind::Local;
  Gate gate;  // physical, sorted targets and matching matrix (Local / RankBlock)
  std::vector<std::pair<int, int>> swaps;  // (global position >= n_local, local position < n_local)
  int source_gate = -1;                    // index in the fused circuit
};

struct ShardPlan {
  int n = 0, n_global = 0, n_local = 0;
  std::vector<ShardOp> ops;
  std::vector<int> final_pos;  // logical qubit -> physical position after the last op
  uint64_t swap_count = 0;     // single-qubit swaps
  uint64_t rank_block_count = 0;
};

// zero_tol as in plan_kernel: entries whose two scalars classify Zero count
// as structural zeros when testing block-diagonality.
ShardPlan plan_sharded(const Circuit& fused, int n_global, double zero_tol = 1e-8, double one_tol = 1e-8);

// The local sub-gate rank `rank` applies for a RankBlock op.  Returns a gate
// with k >= 1 local targets, or a 0-qubit "scalar" gate (targets empty, 1x1
// matrix) when every target is global.
Gate rank_subgate(const ShardOp& op, int n_local, uint64_t rank);

// Physical index of logical basis state `x` under `pos` (logical -> physical).
uint64_t physical_index(uint64_t x, const std::vector<int>& pos);

}  // namespace tilesim
