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
//   Swap       exchange global positions with local ones, all pairs of one
//              gate at once: the bit transpositions (G_i <-> L_i) form an
//              involution of the physical index, applied in place over peer
//              memory -- one grouped all-to-all among the ranks that differ
//              in the G_i bits (each rank keeps 2^-m of its shard)
//
// Pipelining: the top `pipeline_bits` local positions T cut a shard into
// 2^pipeline_bits slabs.  When the swap leaves T alone, the gates right after
// it that never touch T (ShardOp::pipeline_ops of them) run slab by slab: the
// exchange of slab c overlaps those gates on slab c - 1; the rest of the
// segment runs on the whole shard once the exchange is complete.  The planner
// avoids T when it picks the local half of a swap.
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
  int pipeline_bits = 0;                   // Swap: slabs (2^bits) the exchange and the next gates pipeline over
  int pipeline_ops = 0;                    // Swap: how many of the following ops run slab by slab
};

struct ShardPlan {
  int n = 0, n_global = 0, n_local = 0;
  std::vector<ShardOp> ops;
  std::vector<int> final_pos;  // logical qubit -> physical position after the last op
  uint64_t swap_count = 0;     // single-qubit swaps
  uint64_t swap_ops = 0;       // exchanges (grouped all-to-alls)
  uint64_t rank_block_count = 0;
  uint64_t pipelined_swaps = 0;
  double zero_tol = 1e-8, one_tol = 1e-8;  // classification used by the planner; executors plan with the same
  int pipeline_bits = 0;                   // T = top pipeline_bits local positions
};

// zero_tol as in plan_kernel: entries whose two scalars classify Zero count
// as structural zeros when testing block-diagonality.  pipeline_bits: see
// above (0 disables; clamped so a slab keeps >= 2^13 amplitudes).
ShardPlan plan_sharded(const Circuit& fused, int n_global, double zero_tol = 1e-8, double one_tol = 1e-8,
                       int pipeline_bits = 2);

// The local sub-gate rank `rank` applies for a RankBlock op.  Returns a gate
// with k >= 1 local targets, or a 0-qubit "scalar" gate (targets empty, 1x1
// matrix) when every target is global.
Gate rank_subgate(const ShardOp& op, int n_local, uint64_t rank);

// Physical index of logical basis state `x` under `pos` (logical -> physical).
uint64_t physical_index(uint64_t x, const std::vector<int>& pos);

}  // namespace tilesim
