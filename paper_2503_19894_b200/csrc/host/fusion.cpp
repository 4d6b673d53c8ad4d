// CircuitTile and the agglomerative fusion pass (SPEC.md:200-405,
// PAPER.md:225-363), plus cost-model persistence and interpolation.
// Pinned semantics, identical to oracle/oracle.cpp:
//  * traverse: rows top to bottom.  Consecutive phase, columns ascending: a
//    block whose cells one row below are all vacant moves down and is not
//    tested this step; otherwise it is tested against the block directly
//    below in that column.  Then the commuting phase tests horizontally
//    adjacent distinct blocks of the same row (smaller min-wire = first).
//    Each (block, block) pair is tested at most once per traversal.
//  * fuse placement: row r+1 if vacant on the union, else row r, else a new
//    row inserted between r and r+1.  Constituent gates = first ++ second.
//  * compress: bottom-up move-down sweeps to a fixed point, drop empty rows.
//  * flatten: rows top to bottom, ascending min-wire; fused matrix = left
//    fold of fuse_matrices over the constituent gates.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <fstream>
#include <set>
#include <sstream>

#include "tilesim/fusion.hpp"

namespace tilesim {

// ------------------------------------------------------------ cost model
std::string serialize_cost_model(const CostModel& cm) {
  std::ostringstream os;
  os.precision(17);
  os << "version 1\nprecision " << cm.precision << "\nbench_n " << cm.bench_n << "\nhost " << cm.host << "\n";
  for (const CostRecord& r : cm.records)
    os << "k=" << r.k << " ops=" << r.op_count << " threads=" << r.threads << " spg=" << r.seconds_per_group << "\n";
  return os.str();
}

CostModel parse_cost_model(const std::string& text) {
  CostModel cm;
  std::istringstream in(text);
  std::string line;
  bool versioned = false;
  for (int ln = 1; std::getline(in, line); ++ln) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ls(line);
    std::string key;
    if (!(ls >> key)) continue;
    if (key == "version") {
      int v = 0;
      if (!(ls >> v) || v != 1) throw ParseError("unsupported cost-model version", ln);
      versioned = true;
    } else if (key == "precision") {
      ls >> cm.precision;
      if (cm.precision != "f64" && cm.precision != "f32") throw ParseError("precision must be f64 or f32", ln);
    } else if (key == "bench_n") {
      ls >> cm.bench_n;
    } else if (key == "host") {
      std::getline(ls, cm.host);
      cm.host.erase(0, cm.host.find_first_not_of(" \t") == std::string::npos ? cm.host.size()
                                                                               : cm.host.find_first_not_of(" \t"));
    } else if (key.rfind("k=", 0) == 0) {
      CostRecord r;
      unsigned long long ops = 0;
      if (std::sscanf(line.c_str(), " k=%d ops=%llu threads=%d spg=%lf", &r.k, &ops, &r.threads,
                      &r.seconds_per_group) != 4)
        throw ParseError("malformed cost record", ln);
      r.op_count = ops;
      if (!(r.seconds_per_group > 0.0)) throw ParseError("seconds_per_group must be positive", ln);
      cm.records.push_back(r);
    } else {
      throw ParseError("unknown cost-model key '" + key + "'", ln);
    }
  }
  if (!versioned) throw ParseError("cost model missing 'version 1' header");
  return cm;
}

void save_cost_model(const CostModel& cm, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw SimError("cannot write cost model: " + path);
  out << serialize_cost_model(cm);
}

CostModel load_cost_model(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cost model file not found: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return parse_cost_model(ss.str());
}

std::optional<double> estimate_cost(const CostModel& cm, int k, uint64_t ops, int threads, int n) {
  std::vector<std::pair<double, double>> knots;  // (log2 ops, spg), first record per ops value
  std::set<uint64_t> seen;
  for (const CostRecord& r : cm.records)
    if (r.k == k && r.threads == threads && seen.insert(r.op_count).second)
      knots.emplace_back(std::log2(static_cast<double>(std::max<uint64_t>(r.op_count, 1))), r.seconds_per_group);
  if (knots.empty()) return std::nullopt;
  std::stable_sort(knots.begin(), knots.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  const double x = std::log2(static_cast<double>(std::max<uint64_t>(ops, 1)));
  double spg = knots.front().second;
  if (x >= knots.back().first) {
    spg = knots.back().second;
  } else if (x > knots.front().first) {
    size_t i = 0;
    while (!(knots[i].first <= x && x <= knots[i + 1].first)) ++i;
    const double f = (x - knots[i].first) / (knots[i + 1].first - knots[i].first);
    spg = knots[i].second + (knots[i + 1].second - knots[i].second) * f;
  }
  return spg * std::ldexp(1.0, n - k);
}

FusionConfig paper_cpu_preset() {
  FusionConfig c;
  c.k_max = 7;
  c.max_op_count = 4096;
  c.mode = FusionMode::Adaptive;
  return c;
}

bool fusible_size_only(const std::vector<int>& a, const std::vector<int>& b, int k) {
  return static_cast<int>(wire_union(a, b).size()) <= k;
}

// ------------------------------------------------------------------ tile
CircuitTile::CircuitTile(const Circuit& source, FusionConfig cfg, const CostModel* cm)
    : src_(source), cfg_(cfg), cm_(cm), n_(source.n_qubits) {}

size_t CircuitTile::slot_of(int id) const {
  if (id < 0 || id >= static_cast<int>(blocks_.size()) || row_of_[id] < 0) throw SimError("tile: dead block id");
  return static_cast<size_t>(id);
}

bool CircuitTile::vacant(int row, const std::vector<int>& wires) const {
  for (int q : wires)
    if (cells_[row][q] >= 0) return false;
  return true;
}

void CircuitTile::place(int row, int id) {
  for (int q : blocks_[id].wires) cells_[row][q] = id;
  row_of_[id] = row;
}

void CircuitTile::lift(int id) {
  for (int q : blocks_[id].wires) cells_[row_of_[id]][q] = -1;
}

void CircuitTile::append_block(const std::vector<int>& gate_indices) {
  GateBlock b;
  b.id = next_id_++;
  b.gates = gate_indices;
  for (int gi : gate_indices) b.wires = wire_union(b.wires, src_.gates[gi].targets);
  // uppermost row below every occupied cell on the block's wires
  int row = 0;
  for (int r = rows() - 1; r >= 0 && row == 0; --r)
    for (int q : b.wires)
      if (cells_[r][q] >= 0) {
        row = r + 1;
        break;
      }
  while (rows() <= row) cells_.emplace_back(n_, -1);
  blocks_.push_back(std::move(b));
  row_of_.push_back(-1);
  place(row, next_id_ - 1);
}

bool CircuitTile::move_block_down(int id, int row) {
  if (row + 1 >= rows() || !vacant(row + 1, blocks_[id].wires)) return false;
  lift(id);
  place(row + 1, id);
  return true;
}

void CircuitTile::materialize(GateBlock& b) {
  if (b.materialized) return;
  Gate acc = src_.gates[b.gates[0]];
  for (size_t i = 1; i < b.gates.size(); ++i) acc = fuse_matrices(acc, src_.gates[b.gates[i]]);
  b.fused = std::move(acc);
  b.materialized = true;
}

int64_t CircuitTile::ops_of(GateBlock& b) {
  if (b.ops < 0) {
    materialize(b);
    b.ops = static_cast<int64_t>(sparsity_profile(b.fused.matrix, cfg_.zero_tol, cfg_.one_tol).op_count);
  }
  return b.ops;
}

// Global qubits (>= n - n_global) a gate acts on non-block-diagonally: some
// nonzero entry (zero_tol) differs between row and column in that bit.
static int global_mixed(const Gate& g, int n, int n_global, double zt, double ot) {
  int count = 0;
  const uint64_t D = g.matrix.dim();
  for (int b = 0; b < g.k(); ++b) {
    if (g.targets[b] < n - n_global) continue;
    bool mixes = false;
    for (uint64_t r = 0; r < D && !mixes; ++r)
      for (uint64_t c = 0; c < D && !mixes; ++c) {
        if (!(((r ^ c) >> b) & 1u)) continue;
        const cplx& v = g.matrix.at(r, c);
        mixes = classify_scalar(v.real(), zt, ot) != ScalarKind::Zero || classify_scalar(v.imag(), zt, ot) != ScalarKind::Zero;
      }
    count += mixes;
  }
  return count;
}

bool CircuitTile::fusible(int first, int second, int k, Gate* product) {
  GateBlock& a = blocks_[first];
  GateBlock& b = blocks_[second];
  if (!fusible_size_only(a.wires, b.wires, k)) return false;
  if (cfg_.mode != FusionMode::Adaptive && cfg_.n_global <= 0) return true;
  // fusible_adaptive: the fused profile is taken on the
  // materialized product = fold(first.gates ++ second.gates).
  materialize(a);
  Gate p = a.fused;
  for (int gi : b.gates) p = fuse_matrices(p, src_.gates[gi]);
  if (cfg_.n_global > 0) {
    materialize(b);
    const int gp = global_mixed(p, n_, cfg_.n_global, cfg_.zero_tol, cfg_.one_tol);
    const int ga = global_mixed(a.fused, n_, cfg_.n_global, cfg_.zero_tol, cfg_.one_tol);
    const int gb = global_mixed(b.fused, n_, cfg_.n_global, cfg_.zero_tol, cfg_.one_tol);
    if (gp > std::max(ga, gb)) return false;
    if (cfg_.mode != FusionMode::Adaptive) {
      *product = std::move(p);
      return true;
    }
  }
  const uint64_t ops = sparsity_profile(p.matrix, cfg_.zero_tol, cfg_.one_tol).op_count;
  if (cfg_.max_op_count && ops > *cfg_.max_op_count) return false;
  if (!cm_) throw ConfigError("adaptive fusion needs a cost model");
  const auto cf = estimate_cost(*cm_, p.k(), ops, cfg_.threads, n_);
  const auto ca = estimate_cost(*cm_, static_cast<int>(a.wires.size()), ops_of(a), cfg_.threads, n_);
  const auto cb = estimate_cost(*cm_, static_cast<int>(b.wires.size()), ops_of(b), cfg_.threads, n_);
  if (!cf || !ca || !cb) return false;  // outside the benchmarked table
  if (!(*cf <= *ca + *cb)) return false;
  *product = std::move(p);
  return true;
}

void CircuitTile::fuse_blocks(int first, int second, int row, Gate* product) {
  GateBlock c;
  c.id = next_id_++;
  c.gates = blocks_[first].gates;
  c.gates.insert(c.gates.end(), blocks_[second].gates.begin(), blocks_[second].gates.end());
  c.wires = wire_union(blocks_[first].wires, blocks_[second].wires);
  if (product && product->k() > 0) {
    c.fused = std::move(*product);
    c.materialized = true;
  }
  lift(first);
  lift(second);
  row_of_[first] = row_of_[second] = -1;
  blocks_[first].fused = Gate{};
  blocks_[second].fused = Gate{};
  blocks_.push_back(std::move(c));
  row_of_.push_back(-1);
  const int id = next_id_ - 1;
  const std::vector<int>& w = blocks_[id].wires;
  if (row + 1 < rows() && vacant(row + 1, w)) {
    place(row + 1, id);
  } else if (vacant(row, w)) {
    place(row, id);
  } else {
    cells_.insert(cells_.begin() + row + 1, std::vector<int>(n_, -1));
    for (int& r : row_of_)
      if (r > row) ++r;
    place(row + 1, id);
  }
}

void CircuitTile::compress() {
  for (bool moved = true; moved;) {
    moved = false;
    for (int r = rows() - 2; r >= 0; --r)
      for (int q = 0; q < n_; ++q) {
        const int id = cells_[r][q];
        if (id >= 0 && blocks_[id].wires.front() == q && move_block_down(id, r)) moved = true;
      }
  }
  std::vector<std::vector<int>> kept;
  for (auto& row : cells_)
    if (std::any_of(row.begin(), row.end(), [](int v) { return v >= 0; })) kept.push_back(std::move(row));
  cells_.swap(kept);
  for (int r = 0; r < rows(); ++r)
    for (int q = 0; q < n_; ++q)
      if (cells_[r][q] >= 0) row_of_[cells_[r][q]] = r;
}

bool CircuitTile::traverse(int k) {
  bool changed = false;
  std::set<std::pair<int, int>> tested;
  for (int r = 0; r < rows(); ++r) {
    for (int q = 0; q < n_ && r < rows(); ++q) {  // consecutive fusion
      const int top = cells_[r][q];
      if (top < 0 || r + 1 >= rows()) continue;
      if (move_block_down(top, r)) continue;
      const int bot = cells_[r + 1][q];
      if (bot < 0 || !tested.insert({top, bot}).second) continue;
      Gate prod;
      if (fusible(top, bot, k, &prod)) {
        fuse_blocks(top, bot, r, &prod);
        changed = true;
      }
    }
    for (int q = 1; q < n_ && r < rows(); ++q) {  // commuting fusion
      const int a = cells_[r][q - 1], b = cells_[r][q];
      if (a < 0 || b < 0 || a == b || !tested.insert({std::min(a, b), std::max(a, b)}).second) continue;
      const bool a_first = blocks_[a].wires.front() < blocks_[b].wires.front();
      const int first = a_first ? a : b, second = a_first ? b : a;
      Gate prod;
      if (fusible(first, second, k, &prod)) {
        fuse_blocks(first, second, r, &prod);
        changed = true;
      }
    }
  }
  compress();
  return changed;
}

Circuit CircuitTile::flatten() {
  Circuit out;
  out.n_qubits = n_;
  for (int r = 0; r < rows(); ++r)
    for (int q = 0; q < n_; ++q) {
      const int id = cells_[r][q];
      if (id < 0 || blocks_[id].wires.front() != q) continue;
      GateBlock& b = blocks_[id];
      if (b.gates.size() == 1) {
        out.gates.push_back(src_.gates[b.gates[0]]);
      } else {
        materialize(b);
        Gate g = b.fused;
        g.name.clear();
        g.params.clear();
        out.gates.push_back(std::move(g));
      }
    }
  return out;
}

std::string CircuitTile::debug_string() const {
  std::ostringstream os;
  for (const auto& row : cells_) {
    for (int q = 0; q < n_; ++q) os << (q ? " " : "") << (row[q] < 0 ? "." : std::to_string(row[q]));
    os << "\n";
  }
  std::set<int> ids;
  for (const auto& row : cells_)
    for (int v : row)
      if (v >= 0) ids.insert(v);
  for (int id : ids) {
    os << id << ":";
    const GateBlock& b = blocks_[id];
    for (size_t i = 0; i < b.gates.size(); ++i) {
      const Gate& g = src_.gates[b.gates[i]];
      os << (i ? " @ " : " ") << (g.name.empty() ? "matrix" : g.name);
      for (int t : g.targets) os << "," << t;
    }
    os << "\n";
  }
  return os.str();
}

CircuitTile build_tile(const Circuit& c, const FusionConfig& cfg, const CostModel* cm) {
  CircuitTile t(c, cfg, cm);
  for (int i = 0; i < static_cast<int>(c.gates.size()); ++i) t.append_block({i});
  return t;
}

Circuit run_fusion(const Circuit& c, const FusionConfig& cfg, const CostModel* cm, FusionStats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  if (cfg.k_max < 1 || cfg.k_max > kFusedQubitCap) throw ConfigError("k_max must be in [1, 12]");
  if (cfg.max_traversals < 1) throw ConfigError("max_traversals must be >= 1");
  if (cfg.mode == FusionMode::Adaptive && !cm) throw ConfigError("adaptive fusion needs a cost model");
  Circuit out;
  if (cfg.mode == FusionMode::None) {
    out = c;
  } else {
    CircuitTile tile = build_tile(c, cfg, cm);
    for (int k = cfg.agglomerative ? std::min(2, cfg.k_max) : cfg.k_max; k <= cfg.k_max; ++k)
      for (int pass = 0; pass < cfg.max_traversals; ++pass)
        if (!tile.traverse(k) || !cfg.multi_traversal) break;
    out = tile.flatten();
  }
  if (stats) {
    stats->original_gate_count = c.gates.size();
    stats->fused_block_count = out.gates.size();
    stats->compression_ratio =
        out.gates.empty() ? 1.0 : static_cast<double>(c.gates.size()) / static_cast<double>(out.gates.size());
    stats->total_op_count = 0;
    for (const Gate& g : out.gates) stats->total_op_count += sparsity_profile(g.matrix, cfg.zero_tol, cfg.one_tol).op_count;
    stats->fusion_wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return out;
}

}  // namespace tilesim
