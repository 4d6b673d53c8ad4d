// Shard planner: logical gates -> per-rank schedule of local applications,
// rank-selected sub-blocks and global/local qubit swaps (tilesim/shard.hpp).
#include <algorithm>

#include "tilesim/shard.hpp"

namespace tilesim {

namespace {

bool structural_zero(const cplx& v, double zt, double ot) {
  return classify_scalar(v.real(), zt, ot) == ScalarKind::Zero && classify_scalar(v.imag(), zt, ot) == ScalarKind::Zero;
}

// gate on the given physical positions (listed in the gate's logical target
// order), re-expressed with sorted physical targets
Gate to_physical(const Gate& g, const std::vector<int>& pos) {
  std::vector<int> args;
  for (int q : g.targets) args.push_back(pos[q]);
  return make_gate_arg_order(g.matrix, args);
}

}  // namespace

uint64_t physical_index(uint64_t x, const std::vector<int>& pos) {
  uint64_t p = 0;
  for (size_t q = 0; q < pos.size(); ++q) p |= ((x >> q) & 1u) << pos[q];
  return p;
}

ShardPlan plan_sharded(const Circuit& fused, int n_global, double zt, double ot, int pipeline_bits) {
  const int n = fused.n_qubits;
  if (n_global < 0 || n_global >= n) throw ConfigError("n_global must be in [0, n)");
  ShardPlan plan;
  plan.n = n;
  plan.n_global = n_global;
  plan.n_local = n - n_global;
  plan.zero_tol = zt;
  plan.one_tol = ot;
  const int nl = plan.n_local;
  if (pipeline_bits < 0) throw ConfigError("pipeline_bits must be >= 0");
  plan.pipeline_bits = n_global == 0 ? 0 : std::max(0, std::min(pipeline_bits, nl - 13));
  const int t_lo = nl - plan.pipeline_bits;  // T = [t_lo, nl)
  std::vector<int> pos(n), at(n);  // logical -> physical, physical -> logical
  for (int q = 0; q < n; ++q) pos[q] = at[q] = q;
  // next use of each logical qubit after gate gi (Belady eviction for swaps)
  std::vector<std::vector<size_t>> uses(n);
  for (size_t gi = 0; gi < fused.gates.size(); ++gi)
    for (int q : fused.gates[gi].targets) uses[q].push_back(gi);
  auto next_use = [&](int q, size_t gi) {
    const auto it = std::upper_bound(uses[q].begin(), uses[q].end(), gi);
    return it == uses[q].end() ? fused.gates.size() + 1 : *it;
  };

  for (size_t gi = 0; gi < fused.gates.size(); ++gi) {
    const Gate& g = fused.gates[gi];
    if (g.k() > nl) throw ConfigError("gate wider than the local qubit count of a shard");
    Gate pg = to_physical(g, pos);
    const uint64_t D = pg.matrix.dim();
    uint64_t gmask = 0;  // local bit index (within the gate) of global targets
    for (int b = 0; b < pg.k(); ++b)
      if (pg.targets[b] >= nl) gmask |= uint64_t{1} << b;
    if (gmask == 0) {
      ShardOp op;
      op.kind = ShardOp::Kind::Local;
      op.gate = std::move(pg);
      op.source_gate = static_cast<int>(gi);
      plan.ops.push_back(std::move(op));
      continue;
    }
    bool block_diag = true;
    for (uint64_t r = 0; r < D && block_diag; ++r)
      for (uint64_t c = 0; c < D && block_diag; ++c)
        if (((r ^ c) & gmask) && !structural_zero(pg.matrix.at(r, c), zt, ot)) block_diag = false;
    if (block_diag) {
      ShardOp op;
      op.kind = ShardOp::Kind::RankBlock;
      op.gate = std::move(pg);
      op.source_gate = static_cast<int>(gi);
      plan.ops.push_back(std::move(op));
      ++plan.rank_block_count;
      continue;
    }
    // bring every global target local: evict the free local qubit whose next
    // use is furthest away (Belady); ties go to the highest position, whose
    // exchanged half is contiguous
    std::vector<int> used;
    for (int q : g.targets) used.push_back(pos[q]);
    ShardOp sw;
    sw.kind = ShardOp::Kind::Swap;
    for (int q : g.targets) {
      if (pos[q] < nl) continue;
      int best = -1;
      size_t best_use = 0;
      bool best_in_t = true;
      for (int cand = nl - 1; cand >= 0; --cand) {
        if (std::find(used.begin(), used.end(), cand) != used.end()) continue;
        const size_t u = next_use(at[cand], gi);
        const bool in_t = cand >= t_lo;
        // outside the pipeline slab bits T first, then furthest next use
        if (best < 0 || (best_in_t && !in_t) || (in_t == best_in_t && u > best_use)) {
          best = cand;
          best_use = u;
          best_in_t = in_t;
        }
      }
      if (best < 0) throw ConfigError("no free local qubit to swap with");
      const int gp = pos[q], lp = best;
      sw.swaps.emplace_back(gp, lp);
      const int lq = at[lp];
      std::swap(pos[q], pos[lq]);
      at[gp] = lq;
      at[lp] = q;
      used.push_back(lp);
    }
    plan.swap_count += sw.swaps.size();
    ++plan.swap_ops;
    plan.ops.push_back(std::move(sw));
    ShardOp op;
    op.kind = ShardOp::Kind::Local;
    op.gate = to_physical(g, pos);
    op.source_gate = static_cast<int>(gi);
    plan.ops.push_back(std::move(op));
  }
  plan.final_pos = pos;
  // which exchanges can pipeline with the segment that follows them
  if (plan.pipeline_bits > 0)
    for (size_t i = 0; i < plan.ops.size(); ++i) {
      ShardOp& sw = plan.ops[i];
      if (sw.kind != ShardOp::Kind::Swap) continue;
      bool ok = true;
      for (const auto& pr : sw.swaps) ok = ok && pr.second < t_lo;
      if (!ok) continue;
      // the prefix of the following segment whose gates keep off T runs slab by slab
      int prefix = 0;
      for (size_t j = i + 1; j < plan.ops.size() && plan.ops[j].kind != ShardOp::Kind::Swap; ++j) {
        bool off_t = true;
        for (int t : plan.ops[j].gate.targets) off_t = off_t && (t >= nl || t < t_lo);
        if (!off_t) break;
        ++prefix;
      }
      if (prefix > 0) {
        sw.pipeline_bits = plan.pipeline_bits;
        sw.pipeline_ops = prefix;
        ++plan.pipelined_swaps;
      }
    }
  return plan;
}

Gate rank_subgate(const ShardOp& op, int n_local, uint64_t rank) {
  const Gate& g = op.gate;
  std::vector<int> lbits, ltargets;
  uint64_t fixed = 0;  // gate-local index bits fixed by the rank
  for (int b = 0; b < g.k(); ++b) {
    if (g.targets[b] >= n_local) fixed |= ((rank >> (g.targets[b] - n_local)) & 1u) << b;
    else {
      lbits.push_back(b);
      ltargets.push_back(g.targets[b]);
    }
  }
  const int kl = static_cast<int>(lbits.size());
  GateMatrix m(kl);
  for (uint64_t r = 0; r < m.dim(); ++r)
    for (uint64_t c = 0; c < m.dim(); ++c) {
      uint64_t rr = fixed, cc = fixed;
      for (int b = 0; b < kl; ++b) {
        rr |= ((r >> b) & 1u) << lbits[b];
        cc |= ((c >> b) & 1u) << lbits[b];
      }
      m.at(r, c) = g.matrix.at(rr, cc);
    }
  Gate out;
  out.matrix = std::move(m);
  out.targets = std::move(ltargets);
  return out;
}

}  // namespace tilesim
