// tilesim -- command-line front door of the B200 path.
//
//   tilesim run <circuit.qc> [flags]       parse -> fuse -> simulate on the GPU -> RunReport
//   tilesim fuse <circuit.qc> -o <out.qc>  fused circuit (blocks as matrix stanzas) + FusionStats
//   tilesim gen <kind> -n N [-d D] [--seed S] -o <out.qc>
//   tilesim costmodel [--bench-n N] [--k-max K] -o <out.cm>   bench_cost_model on the GPU
//
// Everything goes through the C ABI (include/tilesim_cuda.h), exactly as an
// FFI caller of the reference would.  Exit codes: 0 ok, 1 parse, 2 config,
// 3 runtime; messages on stderr.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "tilesim_cuda.h"

namespace {

struct CliError {
  int code;
  std::string msg;
};

void check(int rc) {
  if (rc != TSG_OK) throw CliError{rc, tsg_last_error()};
}

struct CliConfig {
  std::string precision = "f64";
  int simd = 0;
  std::string fusion = "size-only";  // none | size-only | adaptive | paper-cpu
  int k_max = 5;
  int64_t max_op_count = -1;
  double zero_tol = 1e-8, one_tol = 1e-8;
  int agglomerative = 1, multi_traversal = 1;
  int threads = static_cast<int>(std::thread::hardware_concurrency());
  std::string cost_model, report, dump_state, output, init = "zero";
  uint64_t seed = 0;
  int n = 0, depth = 1;
  int bench_n = 28, bench_k_max = 6, repetitions = 5;
  int device = 0;
};

const char* kHelp =
    "usage: tilesim <command> [args] [flags]\n"
    "commands:\n"
    "  run <circuit.qc>          parse, fuse, simulate on the GPU, print the RunReport\n"
    "  fuse <circuit.qc>         write the fused circuit (-o) and print FusionStats\n"
    "  gen <kind>                write a benchmark circuit (qft ala rqc qvc iqp hes qaoa)\n"
    "  costmodel                 benchmark the GPU kernels into a cost-model file (-o)\n"
    "flags (defaults):\n"
    "  --precision f32|f64       state precision (f64)\n"
    "  -S, --simd N              SIMD exponent s; the GPU kernels use s = 0 (0)\n"
    "  --fusion MODE             none | size-only | adaptive | paper-cpu (size-only)\n"
    "  --k-max N                 largest fused block (5)\n"
    "  --max-op-count N          op-count cap of a fused block (unset)\n"
    "  --zero-tolerance X        Zero classification tolerance (1e-8)\n"
    "  --one-tolerance X         +-1 classification tolerance (1e-8)\n"
    "  --agglomerative 0|1       fuse k = 2..k_max in turn (1)\n"
    "  --multi-traversal 0|1     repeat traversals to a fixed point (1)\n"
    "  --threads N               cost-model thread column (host logical cores)\n"
    "  --cost-model PATH         cost model for adaptive fusion\n"
    "  --report PATH             key=value RunReport / FusionStats file\n"
    "  --dump-state PATH         QSV1 amplitude dump after run\n"
    "  --init zero|basis:X|random:SEED   initial state of run (zero)\n"
    "  -o, --output PATH         output file of fuse / gen / costmodel\n"
    "  -n N, -d/--depth D, --seed S      gen parameters (depth 1, seed 0)\n"
    "  --bench-n N, --bench-k-max K, --repetitions R   costmodel parameters (28, 6, 5)\n"
    "  --device N                CUDA device (0)\n";

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw CliError{TSG_ERR_PARSE, "cannot read " + path};
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void write_file(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw CliError{TSG_ERR_CONFIG, "cannot write " + path};
  f << text;
}

std::string serialize(const tsc_circuit* c) {
  size_t need = 0;
  check(tsc_serialize_circuit(c, nullptr, 0, &need));
  std::string s(need, '\0');
  check(tsc_serialize_circuit(c, s.data(), s.size(), &need));
  s.resize(need - 1);
  return s;
}

tsc_fusion_config fusion_config(const CliConfig& c) {
  tsc_fusion_config f{};
  f.mode = c.fusion == "none" ? 0 : (c.fusion == "adaptive" || c.fusion == "paper-cpu" ? 2 : 1);
  if (c.fusion != "none" && c.fusion != "size-only" && c.fusion != "adaptive" && c.fusion != "paper-cpu")
    throw CliError{TSG_ERR_CONFIG, "unknown fusion mode " + c.fusion};
  f.k_max = c.fusion == "paper-cpu" ? 7 : c.k_max;
  f.max_op_count = c.fusion == "paper-cpu" ? 4096 : c.max_op_count;
  f.agglomerative = c.agglomerative;
  f.multi_traversal = c.multi_traversal;
  f.zero_tol = c.zero_tol;
  f.one_tol = c.one_tol;
  f.max_traversals = 64;
  f.threads = c.threads;
  return f;
}

// fused circuit + stats; the caller destroys the circuit
tsc_circuit* fuse(const tsc_circuit* c, const CliConfig& cfg, tsc_fusion_stats* st) {
  tsc_cost_model* cm = nullptr;
  if (!cfg.cost_model.empty()) check(tsc_cost_model_parse(read_file(cfg.cost_model).c_str(), &cm));
  const tsc_fusion_config fc = fusion_config(cfg);
  if (fc.mode == 2 && !cm) throw CliError{TSG_ERR_CONFIG, "adaptive fusion needs --cost-model"};
  tsc_circuit* out = nullptr;
  const int rc = tsc_run_fusion(c, &fc, cm, &out, st);
  if (cm) tsc_cost_model_destroy(cm);
  check(rc);
  return out;
}

std::string stats_kv(const tsc_fusion_stats& s) {
  std::ostringstream o;
  o << "original_gate_count=" << s.original_gate_count << "\nfused_block_count=" << s.fused_block_count
    << "\ntotal_op_count=" << s.total_op_count << "\ncompression_ratio=" << s.compression_ratio
    << "\nfusion_wall_time=" << s.fusion_wall_time << "\n";
  return o.str();
}

int cmd_run(const std::string& path, const CliConfig& cfg) {
  if (cfg.simd != 0) throw CliError{TSG_ERR_CONFIG, "the GPU kernels use the s = 0 group space (PAPER.md:380)"};
  const int bits = cfg.precision == "f32" ? 32 : 64;
  if (cfg.precision != "f32" && cfg.precision != "f64") throw CliError{TSG_ERR_CONFIG, "precision must be f32 or f64"};
  tsc_circuit* c = nullptr;
  check(tsc_parse_circuit(read_file(path).c_str(), &c));
  int n = 0;
  check(tsc_circuit_n_qubits(c, &n));
  tsc_fusion_stats fs{};
  tsc_circuit* fused = fuse(c, cfg, &fs);
  tsg_ctx* ctx = nullptr;
  check(tsg_ctx_create(cfg.device, &ctx));
  tsg_state* sv = nullptr;
  check(tsg_state_create(ctx, n, bits, &sv));
  if (cfg.init == "zero") {
    check(tsg_state_init_zero(sv));
  } else if (cfg.init.rfind("basis:", 0) == 0) {
    check(tsg_state_init_basis(sv, std::strtoull(cfg.init.c_str() + 6, nullptr, 0)));
  } else if (cfg.init.rfind("random:", 0) == 0) {
    check(tsg_state_init_random(sv, std::strtoull(cfg.init.c_str() + 7, nullptr, 0)));
  } else {
    throw CliError{TSG_ERR_CONFIG, "--init must be zero, basis:X or random:SEED"};
  }
  tsg_program* prog = nullptr;
  check(tsg_program_create(ctx, fused, cfg.zero_tol, cfg.one_tol, bits, &prog));
  tsg_run_report rep{};
  check(tsg_program_run(sv, prog, 1, &rep));
  double nrm = 0.0;
  check(tsg_norm(sv, &nrm));
  if (!cfg.dump_state.empty()) check(tsg_state_dump(sv, cfg.dump_state.c_str()));
  std::ostringstream kv;
  kv << "n_qubits=" << n << "\nprecision=" << cfg.precision << "\n" << stats_kv(fs) << "planning_s=" << rep.planning_s
     << "\nexecution_s=" << rep.execution_s << "\ngates=" << rep.gates << "\nlaunches=" << rep.launches
     << "\nbytes=" << rep.bytes << "\ntouched_bytes=" << rep.touched_bytes << "\nhbm_GBps="
     << (rep.execution_s > 0 ? rep.bytes / rep.execution_s / 1e9 : 0.0) << "\nnorm=" << nrm << "\n";
  std::printf("%-22s %s\n", "circuit", path.c_str());
  std::printf("%-22s %d (%s)\n", "qubits", n, cfg.precision.c_str());
  std::printf("%-22s %llu -> %llu (ratio %.2f, %.3f s)\n", "fusion", (unsigned long long)fs.original_gate_count,
              (unsigned long long)fs.fused_block_count, fs.compression_ratio, fs.fusion_wall_time);
  std::printf("%-22s %.6f s planning, %.6f s device\n", "simulation", rep.planning_s, rep.execution_s);
  std::printf("%-22s %llu\n", "kernel launches", (unsigned long long)rep.launches);
  std::printf("%-22s %.12f\n", "norm", nrm);
  if (!cfg.report.empty()) write_file(cfg.report, kv.str());
  tsg_program_destroy(prog);
  tsg_state_destroy(sv);
  tsg_ctx_destroy(ctx);
  tsc_circuit_destroy(fused);
  tsc_circuit_destroy(c);
  return 0;
}

int cmd_fuse(const std::string& path, const CliConfig& cfg) {
  if (cfg.output.empty()) throw CliError{TSG_ERR_CONFIG, "fuse needs -o <out.qc>"};
  tsc_circuit* c = nullptr;
  check(tsc_parse_circuit(read_file(path).c_str(), &c));
  tsc_fusion_stats fs{};
  tsc_circuit* fused = fuse(c, cfg, &fs);
  write_file(cfg.output, serialize(fused));
  std::printf("original=%llu fused=%llu ratio=%.4f\n", (unsigned long long)fs.original_gate_count,
              (unsigned long long)fs.fused_block_count, fs.compression_ratio);
  if (!cfg.report.empty()) write_file(cfg.report, stats_kv(fs));
  tsc_circuit_destroy(fused);
  tsc_circuit_destroy(c);
  return 0;
}

int cmd_gen(const std::string& kind, const CliConfig& cfg) {
  if (cfg.output.empty()) throw CliError{TSG_ERR_CONFIG, "gen needs -o <out.qc>"};
  tsc_circuit* c = nullptr;
  check(tsc_gen_benchmark(kind.c_str(), cfg.n, cfg.depth, cfg.seed, &c));
  write_file(cfg.output, serialize(c));
  tsc_circuit_destroy(c);
  return 0;
}

int cmd_costmodel(const CliConfig& cfg) {
  if (cfg.output.empty()) throw CliError{TSG_ERR_CONFIG, "costmodel needs -o <out.cm>"};
  const int bits = cfg.precision == "f32" ? 32 : 64;
  tsg_ctx* ctx = nullptr;
  check(tsg_ctx_create(cfg.device, &ctx));
  tsc_cost_model* cm = nullptr;
  check(tsg_bench_cost_model(ctx, cfg.bench_n, cfg.bench_k_max, bits, cfg.repetitions, cfg.seed, &cm));
  size_t need = 0;
  check(tsc_cost_model_serialize(cm, nullptr, 0, &need));
  std::string text(need, '\0');
  check(tsc_cost_model_serialize(cm, text.data(), text.size(), &need));
  text.resize(need - 1);
  write_file(cfg.output, text);
  std::printf("%s", text.c_str());
  tsc_cost_model_destroy(cm);
  tsg_ctx_destroy(ctx);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
      std::printf("%s", kHelp);
      return argc < 2 ? 2 : 0;
    }
    const std::string cmd = argv[1];
    CliConfig cfg;
    std::vector<std::string> pos;
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) throw CliError{TSG_ERR_CONFIG, "missing value for " + a};
        return argv[++i];
      };
      auto num = [&](const std::string& v) {
        char* end = nullptr;
        const double x = std::strtod(v.c_str(), &end);
        if (end == v.c_str() || *end) throw CliError{TSG_ERR_CONFIG, "bad number for " + a + ": " + v};
        return x;
      };
      if (a == "--precision") cfg.precision = val();
      else if (a == "-S" || a == "--simd") cfg.simd = static_cast<int>(num(val()));
      else if (a == "--fusion") cfg.fusion = val();
      else if (a == "--k-max") cfg.k_max = static_cast<int>(num(val()));
      else if (a == "--max-op-count") cfg.max_op_count = static_cast<int64_t>(num(val()));
      else if (a == "--zero-tolerance") cfg.zero_tol = num(val());
      else if (a == "--one-tolerance") cfg.one_tol = num(val());
      else if (a == "--agglomerative") cfg.agglomerative = static_cast<int>(num(val()));
      else if (a == "--multi-traversal") cfg.multi_traversal = static_cast<int>(num(val()));
      else if (a == "--threads") cfg.threads = static_cast<int>(num(val()));
      else if (a == "--cost-model") cfg.cost_model = val();
      else if (a == "--report") cfg.report = val();
      else if (a == "--dump-state") cfg.dump_state = val();
      else if (a == "--init") cfg.init = val();
      else if (a == "-o" || a == "--output") cfg.output = val();
      else if (a == "-n") cfg.n = static_cast<int>(num(val()));
      else if (a == "-d" || a == "--depth") cfg.depth = static_cast<int>(num(val()));
      else if (a == "--seed") cfg.seed = static_cast<uint64_t>(num(val()));
      else if (a == "--bench-n") cfg.bench_n = static_cast<int>(num(val()));
      else if (a == "--bench-k-max") cfg.bench_k_max = static_cast<int>(num(val()));
      else if (a == "--repetitions") cfg.repetitions = static_cast<int>(num(val()));
      else if (a == "--device") cfg.device = static_cast<int>(num(val()));
      else if (!a.empty() && a[0] == '-') throw CliError{TSG_ERR_CONFIG, "unknown flag " + a};
      else pos.push_back(a);
    }
    if (cmd == "run" && pos.size() == 1) return cmd_run(pos[0], cfg);
    if (cmd == "fuse" && pos.size() == 1) return cmd_fuse(pos[0], cfg);
    if (cmd == "gen" && pos.size() == 1) return cmd_gen(pos[0], cfg);
    if (cmd == "costmodel" && pos.empty()) return cmd_costmodel(cfg);
    throw CliError{TSG_ERR_CONFIG, "bad command line (see tilesim --help)"};
  } catch (const CliError& e) {
    std::fprintf(stderr, "tilesim: %s\n", e.msg.c_str());
    return e.code;
  }
}
