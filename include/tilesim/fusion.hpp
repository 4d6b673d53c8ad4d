// tilesim/fusion.hpp -- CircuitTile IR, Algorithm 1 traversal, agglomerative
// fusion driver, size-only / adaptive predicates, and the cost model.
//
// SPEC-only in the reference (no shipped code):
//   GateBlock / CircuitTile / build_tile / append_block / traverse /
//   move_block_down / fuse_blocks / compress / flatten
//   FusionConfig / CostRecord / CostModel / FusionStats /
//   run_fusion / fusible_* / estimate_cost / save/load
// Algorithm 1 is PAPER.md:247-310.  Ambiguities are pinned once
// and shared with the oracle so fusion plans compare bit-for-bit.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "tilesim/ir.hpp"

namespace tilesim {

// ------------------------------------------------------------ cost model
struct CostRecord {
  int k = 0;
  uint64_t op_count = 0;
  int threads = 0;  // CPU: worker threads; B200: CTA size of the timed kernel
  double seconds_per_group = 0.0;
};

struct CostModel {
  std::vector<CostRecord> records;
  int bench_n = 0;
  std::string precision = "f64";  // f64 | f32
  std::string host;
};

std::string serialize_cost_model(const CostModel& cm);
CostModel parse_cost_model(const std::string& text);  // throws ParseError
void save_cost_model(const CostModel& cm, const std::string& path);
CostModel load_cost_model(const std::string& path);   // "not found" is a distinct ParseError

// seconds for one application of a k-qubit gate with `ops` on an n-qubit
// state; nullopt when (k, threads) has no records.
std::optional<double> estimate_cost(const CostModel& cm, int k, uint64_t ops, int threads, int n);

// ---------------------------------------------------------------- config
enum class FusionMode { None, SizeOnly, Adaptive };

struct FusionConfig {
  int k_max = 5;
  std::optional<uint64_t> max_op_count;
  FusionMode mode = FusionMode::SizeOnly;
  bool agglomerative = true;
  bool multi_traversal = true;
  double zero_tol = 1e-8, one_tol = 1e-8;
  int max_traversals = 64;
  int threads = 1;  // thread/CTA column used for cost lookups
  // Shard-aware fusion (B200 extension): with the top
  // n_global qubits sharded across GPUs, a fusion is refused when the fused
  // gate mixes (acts non-block-diagonally on) more of those qubits than the
  // wider-mixing of its two parts -- such a product would need an exchange
  // its parts did not.  0: the reference's fusion, unchanged (the default:
  // measured on RQC-33 / TFIM-36 / ALA-30 / IQP-30 over 8 ranks, the
  // restriction leaves more, smaller gates and MORE exchanges -- 4 -> 5,
  // 5 -> 14, 7 -> 9, 1 -> 4).
  int n_global = 0;
};

// Preset "paper-cpu": k_max 7, op cap 4096, adaptive.
FusionConfig paper_cpu_preset();

struct FusionStats {
  uint64_t original_gate_count = 0, fused_block_count = 0, total_op_count = 0;
  double compression_ratio = 1.0, fusion_wall_time = 0.0;
};

// ------------------------------------------------------------------ tile
struct GateBlock {
  int id = -1;
  std::vector<int> gates;  // indices into the source circuit, time order
  std::vector<int> wires;  // sorted union of targets
  bool materialized = false;
  Gate fused;              // valid when materialized
  int64_t ops = -1;        // cached op_count (cfg tolerances), -1 unknown
};

class CircuitTile {
 public:
  CircuitTile(const Circuit& source, FusionConfig cfg, const CostModel* cm = nullptr);

  void append_block(const std::vector<int>& gate_indices);
  bool traverse(int k);               // one pass of Algorithm 1 + compress
  bool move_block_down(int id, int row);
  void compress();
  Circuit flatten();

  int rows() const { return static_cast<int>(cells_.size()); }
  int cell(int row, int q) const { return cells_[row][q]; }
  const GateBlock& block(int id) const { return blocks_.at(slot_of(id)); }
  std::string debug_string() const;   // SPEC.md:299 tile dump

 private:
  bool fusible(int first, int second, int k, Gate* product);
  void fuse_blocks(int first, int second, int row, Gate* product);
  void materialize(GateBlock& b);
  int64_t ops_of(GateBlock& b);
  size_t slot_of(int id) const;
  bool vacant(int row, const std::vector<int>& wires) const;
  void place(int row, int id);
  void lift(int id);

  const Circuit& src_;
  FusionConfig cfg_;
  const CostModel* cm_;
  int n_;
  std::vector<std::vector<int>> cells_;  // block id or -1
  std::vector<GateBlock> blocks_;        // live and dead blocks, indexed by id
  std::vector<int> row_of_;              // by id, -1 when dead
  int next_id_ = 0;
};

CircuitTile build_tile(const Circuit& c, const FusionConfig& cfg, const CostModel* cm = nullptr);

bool fusible_size_only(const std::vector<int>& wires_top, const std::vector<int>& wires_bot, int k);

Circuit run_fusion(const Circuit& c, const FusionConfig& cfg, const CostModel* cm, FusionStats* stats);

}  // namespace tilesim
