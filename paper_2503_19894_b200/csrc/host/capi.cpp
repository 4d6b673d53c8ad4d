// C ABI for the host-only part of the surface: circuit IR, generators, text
// format, fusion pass and cost model (include/tilesim_cuda.h, tsc_*).
#include <atomic>
#include <cstring>

#include "handles.hpp"
#include "rendezvous.hpp"
#include "tilesim/pass.hpp"

namespace tsg_detail {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace tsg_detail

using namespace tilesim;
using tsg_detail::require;

namespace {

GateMatrix matrix_from(int k, const double* m) {
  GateMatrix g(k);
  for (size_t i = 0; i < g.entries().size(); ++i) g.entries()[i] = cplx(m[2 * i], m[2 * i + 1]);
  return g;
}

int copy_out(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap > 0) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return TSG_OK;
}

FusionConfig to_config(const tsc_fusion_config* c) {
  FusionConfig f;
  require(c->mode >= 0 && c->mode <= 2, "fusion mode must be 0 (none), 1 (size-only) or 2 (adaptive)");
  f.mode = c->mode == 0 ? FusionMode::None : (c->mode == 1 ? FusionMode::SizeOnly : FusionMode::Adaptive);
  f.k_max = c->k_max;
  if (c->max_op_count >= 0) f.max_op_count = static_cast<uint64_t>(c->max_op_count);
  f.agglomerative = c->agglomerative != 0;
  f.multi_traversal = c->multi_traversal != 0;
  f.zero_tol = c->zero_tol;
  f.one_tol = c->one_tol;
  f.max_traversals = c->max_traversals;
  f.threads = c->threads;
  f.n_global = c->n_global;
  require(f.n_global >= 0, "n_global must be >= 0");
  require(f.zero_tol >= 0 && f.one_tol >= 0, "tolerances must be >= 0");
  return f;
}

}  // namespace

extern "C" {

const char* tsg_last_error(void) { return tsg_detail::g_last_error.c_str(); }
const char* tsg_version(void) { return "tilesim-b200 0.1 (sm_100a)"; }

int tsc_circuit_create(int n_qubits, tsc_circuit** out) {
  TSG_TRY({
    require(out != nullptr, "null output handle");
    require(n_qubits >= 1 && n_qubits <= 62, "qubit count must be in [1, 62]");
    *out = new tsc_circuit();
    (*out)->c.n_qubits = n_qubits;
  })
}

int tsc_circuit_destroy(tsc_circuit* c) {
  delete c;
  return TSG_OK;
}

int tsc_circuit_copy(const tsc_circuit* c, tsc_circuit** out) {
  TSG_TRY({
    require(c && out, "null handle");
    *out = new tsc_circuit(*c);
  })
}

int tsc_circuit_add_named(tsc_circuit* c, const char* name, const double* params, int n_params, const int* qubits,
                          int n_qubits) {
  TSG_TRY({
    require(c && name, "null handle");
    std::vector<int> q(qubits, qubits + n_qubits);
    for (int x : q)
      if (x < 0 || x >= c->c.n_qubits) throw ConfigError("qubit index out of range");
    c->c.gates.push_back(make_named_gate(name, std::vector<double>(params, params + n_params), q));
  })
}

int tsc_circuit_add_matrix(tsc_circuit* c, int k, const int* qubits, const double* matrix) {
  TSG_TRY({
    require(c && qubits && matrix, "null argument");
    require(k >= 1 && k <= kFusedQubitCap, "matrix gate size must be in [1, 12]");
    std::vector<int> q(qubits, qubits + k);
    for (int x : q)
      if (x < 0 || x >= c->c.n_qubits) throw ConfigError("qubit index out of range");
    c->c.gates.push_back(make_gate_arg_order(matrix_from(k, matrix), q));
  })
}

int tsc_circuit_n_qubits(const tsc_circuit* c, int* out) {
  TSG_TRY({
    require(c && out, "null argument");
    *out = c->c.n_qubits;
  })
}

int tsc_circuit_n_gates(const tsc_circuit* c, uint64_t* out) {
  TSG_TRY({
    require(c && out, "null argument");
    *out = c->c.gates.size();
  })
}

int tsc_circuit_gate(const tsc_circuit* c, uint64_t i, int* k, int* targets, double* matrix) {
  TSG_TRY({
    require(c != nullptr, "null handle");
    require(i < c->c.gates.size(), "gate index out of range");
    const Gate& g = c->c.gates[i];
    if (k) *k = g.k();
    if (targets)
      for (int j = 0; j < g.k(); ++j) targets[j] = g.targets[j];
    if (matrix)
      for (size_t j = 0; j < g.matrix.entries().size(); ++j) {
        matrix[2 * j] = g.matrix.entries()[j].real();
        matrix[2 * j + 1] = g.matrix.entries()[j].imag();
      }
  })
}

const char* tsc_circuit_gate_name(const tsc_circuit* c, uint64_t i) {
  if (!c || i >= c->c.gates.size()) return "";
  return c->c.gates[i].name.c_str();
}

int tsc_gen_benchmark(const char* kind, int n, int depth, uint64_t seed, tsc_circuit** out) {
  TSG_TRY({
    require(kind && out, "null argument");
    *out = new tsc_circuit{gen_benchmark(parse_benchmark_kind(kind), n, depth, seed)};
  })
}

int tsc_parse_circuit(const char* text, tsc_circuit** out) {
  TSG_TRY({
    require(text && out, "null argument");
    *out = new tsc_circuit{parse_circuit(text)};
  })
}

int tsc_serialize_circuit(const tsc_circuit* c, char* buf, size_t cap, size_t* needed) {
  TSG_TRY({
    require(c != nullptr, "null handle");
    copy_out(serialize_circuit(c->c), buf, cap, needed);
  })
}

int tsc_run_fusion(const tsc_circuit* c, const tsc_fusion_config* cfg, const tsc_cost_model* cm, tsc_circuit** out,
                   tsc_fusion_stats* stats) {
  TSG_TRY({
    require(c && cfg && out, "null argument");
    FusionStats st;
    Circuit fused = run_fusion(c->c, to_config(cfg), cm ? &cm->cm : nullptr, &st);
    *out = new tsc_circuit{std::move(fused)};
    if (stats) {
      stats->original_gate_count = st.original_gate_count;
      stats->fused_block_count = st.fused_block_count;
      stats->total_op_count = st.total_op_count;
      stats->compression_ratio = st.compression_ratio;
      stats->fusion_wall_time = st.fusion_wall_time;
    }
  })
}

int tsc_cost_model_parse(const char* text, tsc_cost_model** out) {
  TSG_TRY({
    require(text && out, "null argument");
    *out = new tsc_cost_model{parse_cost_model(text)};
  })
}

int tsc_cost_model_destroy(tsc_cost_model* cm) {
  delete cm;
  return TSG_OK;
}

int tsc_cost_model_serialize(const tsc_cost_model* cm, char* buf, size_t cap, size_t* needed) {
  TSG_TRY({
    require(cm != nullptr, "null handle");
    copy_out(serialize_cost_model(cm->cm), buf, cap, needed);
  })
}

int tsc_estimate_cost(const tsc_cost_model* cm, int k, uint64_t op_count, int threads, int n, double* seconds) {
  TSG_TRY({
    require(cm && seconds, "null argument");
    const auto c = estimate_cost(cm->cm, k, op_count, threads, n);
    if (!c) throw ConfigError("no cost records for this gate size / thread count");
    *seconds = *c;
  })
}

}  // extern "C"

// ---------------------------------------------------------------- sharding
extern "C" {

int tsc_plan_passes(const tsc_circuit* fused, int precision_bits, double zero_tol, double one_tol, int* step_of_gate,
                    int* step_is_pass, int* step_high, uint64_t* n_steps) {
  TSG_TRY({
    require(fused && n_steps, "null argument");
    require(precision_bits == 64 || precision_bits == 32, "precision_bits must be 64 or 32");
    const int n = fused->c.n_qubits;
    std::vector<LaunchStructure> ls;
    for (const Gate& g : fused->c.gates) {
      const KernelPlan plan = plan_kernel(g, n, 0, zero_tol, one_tol, false);
      ls.push_back(precision_bits == 64 ? plan.launch : derive_launch(plan, nullptr, precision_bits));
    }
    const auto steps = plan_passes(ls, n, pass_config(precision_bits, n));
    if (step_of_gate)
      for (size_t g = 0; g < ls.size(); ++g) step_of_gate[g] = -1;
    for (size_t s = 0; s < steps.size(); ++s) {
      if (step_of_gate)
        for (int g : steps[s].gates) step_of_gate[g] = static_cast<int>(s);
      if (step_is_pass) step_is_pass[s] = steps[s].is_pass ? 1 : (steps[s].is_permute ? 2 : 0);
      if (step_high)
        for (int h = 0; h < 16; ++h)
          step_high[16 * s + h] = h < static_cast<int>(steps[s].high.size()) ? steps[s].high[h] : -1;
    }
    *n_steps = steps.size();
  })
}

int tsc_shard_plan_create(const tsc_circuit* fused, int n_global, double zero_tol, double one_tol, int pipeline_bits,
                          tsc_shard_plan** out) {
  TSG_TRY({
    require(fused && out, "null argument");
    static std::atomic<uint64_t> serial{0};
    *out = new tsc_shard_plan{plan_sharded(fused->c, n_global, zero_tol, one_tol, pipeline_bits), ++serial};
  })
}

int tsc_shard_plan_stats(const tsc_shard_plan* p, uint64_t* swap_ops, uint64_t* pipelined_swaps, int* pipeline_bits) {
  TSG_TRY({
    require(p != nullptr, "null handle");
    if (swap_ops) *swap_ops = p->plan.swap_ops;
    if (pipelined_swaps) *pipelined_swaps = p->plan.pipelined_swaps;
    if (pipeline_bits) *pipeline_bits = p->plan.pipeline_bits;
  })
}

int tsc_shard_plan_destroy(tsc_shard_plan* p) {
  delete p;
  return TSG_OK;
}

int tsc_shard_plan_info(const tsc_shard_plan* p, int* n_qubits, int* n_global, uint64_t* n_ops, uint64_t* swaps,
                        uint64_t* rank_blocks) {
  TSG_TRY({
    require(p != nullptr, "null handle");
    if (n_qubits) *n_qubits = p->plan.n;
    if (n_global) *n_global = p->plan.n_global;
    if (n_ops) *n_ops = p->plan.ops.size();
    if (swaps) *swaps = p->plan.swap_count;
    if (rank_blocks) *rank_blocks = p->plan.rank_block_count;
  })
}

static void put_gate(const Gate& g, int* k, int* targets, double* matrix) {
  if (k) *k = g.k();
  if (targets)
    for (int j = 0; j < g.k(); ++j) targets[j] = g.targets[j];
  if (matrix)
    for (size_t j = 0; j < g.matrix.entries().size(); ++j) {
      matrix[2 * j] = g.matrix.entries()[j].real();
      matrix[2 * j + 1] = g.matrix.entries()[j].imag();
    }
}

int tsc_shard_plan_op(const tsc_shard_plan* p, uint64_t i, int* kind, int* k, int* targets, double* matrix,
                      int* n_swaps, int* swap_pairs, int* source_gate, int* pipeline_bits, int* pipeline_ops) {
  TSG_TRY({
    require(p != nullptr, "null handle");
    require(i < p->plan.ops.size(), "op index out of range");
    const ShardOp& op = p->plan.ops[i];
    if (kind) *kind = static_cast<int>(op.kind);
    if (op.kind == ShardOp::Kind::Swap) {
      if (k) *k = 0;
    } else {
      put_gate(op.gate, k, targets, matrix);
    }
    if (n_swaps) *n_swaps = static_cast<int>(op.swaps.size());
    if (swap_pairs)
      for (size_t s = 0; s < op.swaps.size(); ++s) {
        swap_pairs[2 * s] = op.swaps[s].first;
        swap_pairs[2 * s + 1] = op.swaps[s].second;
      }
    if (source_gate) *source_gate = op.source_gate;
    if (pipeline_bits) *pipeline_bits = op.pipeline_bits;
    if (pipeline_ops) *pipeline_ops = op.pipeline_ops;
  })
}

int tsc_shard_rank_subgate(const tsc_shard_plan* p, uint64_t i, uint64_t rank, int* k, int* targets, double* matrix) {
  TSG_TRY({
    require(p != nullptr, "null handle");
    require(i < p->plan.ops.size(), "op index out of range");
    require(p->plan.ops[i].kind == ShardOp::Kind::RankBlock, "op is not a rank block");
    require(rank < (uint64_t{1} << p->plan.n_global), "rank out of range");
    put_gate(rank_subgate(p->plan.ops[i], p->plan.n_local, rank), k, targets, matrix);
  })
}

int tsc_shard_final_pos(const tsc_shard_plan* p, int* pos) {
  TSG_TRY({
    require(p && pos, "null argument");
    for (int q = 0; q < p->plan.n; ++q) pos[q] = p->plan.final_pos[q];
  })
}

int tsg_rendezvous_selftest(const unsigned char id[128], int rank, int world, int iters, uint64_t* checksum) {
  TSG_TRY({
    require(id && checksum, "null argument");
    tilesim::ShmRendezvous rv(id, rank, world, sizeof(uint64_t), 120.0);
    uint64_t sum = 0;
    for (int it = 0; it < iters; ++it) {
      *static_cast<uint64_t*>(rv.slot(rank)) = static_cast<uint64_t>(it) * 1000 + rank;
      rv.barrier();
      for (int r = 0; r < world; ++r) sum += *static_cast<uint64_t*>(rv.slot(r));
      rv.barrier();
    }
    *checksum = sum;
  })
}

}  // extern "C"
