// Tile-pass planning (include/tilesim/pass.hpp).  Host only: the device blob
// for a planned pass is built in cuda/runtime.cu (build_pass_blob).
#include "tilesim/pass.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace tilesim {

bool pass_jit_expected(int n_qubits) {
  const char* off = std::getenv("TSG_PASS_JIT");
  if (off && off[0] == '0' && off[1] == '\0') return false;
  const char* e = std::getenv("TSG_PASS_JIT_MIN_N");
  return n_qubits >= (e ? std::atoi(e) : 24);
}

PassConfig pass_config(int precision_bits, int n_qubits) {
  PassConfig c;
  const bool jit = n_qubits > 0 && pass_jit_expected(n_qubits);
  if (precision_bits == 64) {
    c.tile_log2 = 11;  // 32 KiB of complex128 per tile
    c.run_log2 = 5;    // 256-byte runs per array
    c.max_gen_ks = 4;  // dense ks = 5 complex128 is FP64-bound: own DMMA kernel
    c.amp_real_bytes = 8;
    c.reg_bits = 3;
    // JIT passes keep the interpreter's complex128 table: the per-op micro
    // costs measured lower (profiles/r02/pass_bench_jit_f64.txt), but QFT-30 and
    // RQC-30 planned with them ran slower (76.7 / 395 ms vs 73.3 / 388 ms)
    (void)jit;
  } else {
    c.tile_log2 = 12;
    c.run_log2 = 6;
    c.max_gen_ks = 5;
    c.amp_real_bytes = 4;
    c.reg_bits = 3;  // of 4: register ops mix at most 3 qubits
    c.base_sweeps = 1.28;
    c.diag_sweeps = 0.05;
    const double gen32[6] = {0.0, 0.25, 0.4, 0.7, 1.6, 2.5};
    std::copy(gen32, gen32 + 6, c.gen_sweeps);
    c.perm_sweeps_reg = 0.45;
    c.perm_sweeps_smem = 0.6;
    c.standalone_sweeps = 1.1;
    if (jit) {  // JIT passes (r02 scripts/pass_bench.py PB_FORCE=1, profiles/r02/pass_bench_jit_f32.txt)
      c.base_sweeps = 1.04;
      c.diag_sweeps = 0.01;
      const double gen32j[6] = {0.0, 0.05, 0.12, 0.45, 1.1, 2.1};
      std::copy(gen32j, gen32j + 6, c.gen_sweeps);
      c.perm_sweeps_reg = 0.25;
      c.perm_sweeps_smem = 0.5;
    }
  }
  // calibration experiments: TSG_PASS_COSTS="base,diag,g1,g2,g3,g4,g5,max_gen_ks"
  if (const char* e = std::getenv("TSG_PASS_COSTS")) {
    double v[8];
    if (std::sscanf(e, "%lf,%lf,%lf,%lf,%lf,%lf,%lf,%lf", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5], &v[6], &v[7]) == 8) {
      c.base_sweeps = v[0];
      c.diag_sweeps = v[1];
      for (int k = 1; k <= 5; ++k) c.gen_sweeps[k] = v[1 + k];
      c.max_gen_ks = static_cast<int>(v[7]);
    }
  }
  if (const char* e = std::getenv("TSG_PASS_GEOM")) std::sscanf(e, "%d,%d", &c.tile_log2, &c.run_log2);  // planner experiments only
  const char* f = std::getenv("TSG_PASS_FORCE");
  c.force = f && f[0] == '1';
  if (std::getenv("TSG_NO_PERMUTE")) c.min_permute_run = 0;
  return c;
}

namespace {

constexpr int kPassOpRecord = 192;  // sizeof(tsg::PassOp)
constexpr int kThreads = 256;       // tsg::kPassThreads (threads of a k_pass CTA)

}  // namespace

std::vector<int> mixed_bits(const LaunchStructure& ls) {
  const int d = 1 << ls.ks;
  int mixed = 0;
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c)
      if (ls.sub_re[r * d + c] != 0.0 || ls.sub_im[r * d + c] != 0.0) mixed |= r ^ c;
  std::vector<int> out;
  for (int b = 0; b < ls.ks; ++b)
    if ((mixed >> b) & 1) out.push_back(b);
  return out;
}

bool monomial(const LaunchStructure& ls) {
  const int d = 1 << ls.ks;
  for (int r = 0; r < d; ++r) {
    int nz = 0;
    for (int c = 0; c < d; ++c) nz += ls.sub_re[r * d + c] != 0.0 || ls.sub_im[r * d + c] != 0.0;
    if (nz != 1) return false;
  }
  return true;
}

std::vector<LaunchStructure> split_blocks(const LaunchStructure& ls, int precision_bits) {
  if (ls.klass != KernelClass::Direct && ls.klass != KernelClass::Tile) return {ls};
  const std::vector<int> ebits = mixed_bits(ls);
  if (static_cast<int>(ebits.size()) == ls.ks || ebits.empty()) return {ls};
  std::vector<int> bbits;
  for (int b = 0; b < ls.ks; ++b)
    if (std::find(ebits.begin(), ebits.end(), b) == ebits.end()) bbits.push_back(b);
  const int ke = static_cast<int>(ebits.size()), nb = static_cast<int>(bbits.size());
  const int d = 1 << ls.ks, de = 1 << ke;
  const int direct_max = precision_bits == 64 ? 4 : 5;
  std::vector<LaunchStructure> out;
  for (int jb = 0; jb < (1 << nb); ++jb) {
    LaunchStructure s;
    s.controls = ls.controls;
    s.control_values = ls.control_values;
    int base = 0;
    for (int i = 0; i < nb; ++i) {
      const int q = ls.sub_targets[bbits[i]];
      s.controls.push_back(q);
      s.control_values |= static_cast<uint64_t>((jb >> i) & 1) << q;
      base |= ((jb >> i) & 1) << bbits[i];
    }
    std::sort(s.controls.begin(), s.controls.end());
    s.ks = ke;
    for (int b : ebits) s.sub_targets.push_back(ls.sub_targets[b]);
    s.offsets.resize(de);
    std::vector<int> full(de);
    for (int j = 0; j < de; ++j) {
      uint64_t q = 0;
      int f = base;
      for (int b = 0; b < ke; ++b) {
        q |= static_cast<uint64_t>((j >> b) & 1) << s.sub_targets[b];
        f |= ((j >> b) & 1) << ebits[b];
      }
      s.offsets[j] = q;
      full[j] = f;
    }
    s.sub_re.resize(de * de);
    s.sub_im.resize(de * de);
    bool diagonal = true, identity = true;
    for (int r = 0; r < de; ++r)
      for (int c = 0; c < de; ++c) {
        const double re = ls.sub_re[full[r] * d + full[c]], im = ls.sub_im[full[r] * d + full[c]];
        s.sub_re[r * de + c] = re;
        s.sub_im[r * de + c] = im;
        s.nonzero_scalars += (re != 0.0) + (im != 0.0);
        if (r != c && (re != 0.0 || im != 0.0)) diagonal = false;
        if (!(re == (r == c ? 1.0 : 0.0) && im == 0.0)) identity = false;
      }
    if (identity) continue;
    s.klass = diagonal ? KernelClass::Diagonal : (ke <= direct_max ? KernelClass::Direct : KernelClass::Tile);
    s.sparse = s.nonzero_scalars * 4 <= 3 * static_cast<uint64_t>(2 * de * de);
    out.push_back(std::move(s));
  }
  return out;
}

PassRole pass_role(const LaunchStructure& ls, const PassConfig& cfg) {
  switch (ls.klass) {
    case KernelClass::Identity: return PassRole::Standalone;
    case KernelClass::Diagonal: return ls.ks <= 7 ? PassRole::Diag : PassRole::Standalone;
    default: {
      const int ke = static_cast<int>(mixed_bits(ls).size());
      const int kmax = monomial(ls) ? 5 : cfg.max_gen_ks;
      if (ke < 1 || ke > kmax || ls.ks - ke > 8) return PassRole::Standalone;
      if (ke + static_cast<int>(ls.controls.size()) > 15) return PassRole::Standalone;
      return PassRole::Gen;
    }
  }
}

int pass_op_bytes(const LaunchStructure& ls, const PassConfig& cfg) {
  const int cplx = 2 * cfg.amp_real_bytes;
  int data = 0;
  if (ls.klass == KernelClass::Diagonal) {
    // table + identity entry, per-thread index bits; a RUN header may be added
    data = ((((1 << ls.ks) + 1) * cplx + 15) & ~15) + kThreads + kPassOpRecord;
  } else {
    const int ke = static_cast<int>(mixed_bits(ls).size());
    const int d = 1 << ke, blocks = 1 << (ls.ks - ke);
    const int groups = 1 << std::max(0, cfg.tile_log2 - ke);  // upper bound: controls may fall outside the tile
    const int block_bytes = monomial(ls) ? ((4 * d + 15) & ~15) + d * cplx : (d * d + 1) * cplx;
    data = ((4 * d + 15) & ~15) + 4 * kThreads + 4 * std::max(1, groups / kThreads) + 16 + blocks * block_bytes;
  }
  return kPassOpRecord + ((data + 15) & ~15);
}

double pass_op_sweeps(const LaunchStructure& ls, const PassConfig& cfg) {
  if (ls.klass == KernelClass::Diagonal) return cfg.diag_sweeps;
  const int ke = static_cast<int>(mixed_bits(ls).size());
  if (monomial(ls)) return ke <= cfg.reg_bits ? cfg.perm_sweeps_reg : cfg.perm_sweeps_smem;
  return cfg.gen_sweeps[std::min(ke, 5)];
}

double standalone_sweeps(const LaunchStructure& ls, const PassConfig& cfg) {
  double sweeps = cfg.standalone_sweeps;
  if (cfg.amp_real_bytes == 4 && ls.ks >= 4) {
    // complex64 4-5 qubit sub-gates run on the INT8 tensor-core kernel, one
    // group per lane: its cost follows how the lanes' groups spread over the
    // shared-memory banks -- the 32 lanes take the 5 lowest qubits that are
    // neither targets nor controls (scripts/umma_bench.py, B200):
    //   <= 2 lanes per bank 1.1 (ks 5: 1.5) sweeps, 8: 1.7, 16: 2.5
    // and a low contiguous target run from qubit 0 stays on the FP64-widened
    // DMMA product: 2.8
    static const bool old_model = std::getenv("TSG_PASS_C64_FLAT") != nullptr;
    if (!old_model) {
      std::vector<int> busy(ls.sub_targets);
      busy.insert(busy.end(), ls.controls.begin(), ls.controls.end());
      int lane_pos[5], nl = 0;
      for (int q = 0; nl < 5; ++q)
        if (std::find(busy.begin(), busy.end(), q) == busy.end()) lane_pos[nl++] = q;
      int cnt[32] = {0}, deg = 0;
      for (int l = 0; l < 32; ++l) {
        int x = 0;
        for (int b = 0; b < 5; ++b) x |= ((l >> b) & 1) << lane_pos[b];
        deg = std::max(deg, ++cnt[x % 32]);
      }
      const bool low_run = ls.sub_targets[0] == 0 && ls.sub_targets[1] == 1;
      if (low_run) sweeps = 2.8;
      else if (deg >= 16) sweeps = 2.5;
      else if (deg >= 8) sweeps = 1.7;
      else if (deg >= 4) sweeps = 1.3;
      else sweeps = ls.ks >= 5 ? 1.5 : 1.1;
    }
  }
  return sweeps * std::ldexp(1.0, -static_cast<int>(ls.controls.size()));
}

bool qubit_permutation(const LaunchStructure& ls, std::vector<int>* sigma) {
  if (ls.klass == KernelClass::Identity || ls.klass == KernelClass::Diagonal || !ls.controls.empty() || ls.ks < 1)
    return false;
  const int D = 1 << ls.ks;
  if (static_cast<int>(ls.sub_re.size()) != D * D) return false;
  std::vector<int> dest(D, -1);  // column j -> row of its single 1
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      const double re = ls.sub_re[static_cast<size_t>(r) * D + c], im = ls.sub_im[static_cast<size_t>(r) * D + c];
      if (im != 0.0 || (re != 0.0 && re != 1.0)) return false;
      if (re == 1.0) {
        if (dest[c] >= 0) return false;
        dest[c] = r;
      }
    }
  std::vector<int> sg(ls.ks);
  for (int b = 0; b < ls.ks; ++b) {
    const int d = dest[1 << b];
    if (d <= 0 || (d & (d - 1)) != 0) return false;
    sg[b] = __builtin_ctz(static_cast<unsigned>(d));
  }
  for (int j = 0; j < D; ++j) {
    int y = 0;
    for (int b = 0; b < ls.ks; ++b) y |= ((j >> b) & 1) << sg[b];
    if (dest[j] != y) return false;
  }
  bool moves = false;
  for (int b = 0; b < ls.ks; ++b) moves |= sg[b] != b;
  if (!moves) return false;
  if (sigma) *sigma = sg;
  return true;
}

// Qubits a gate touches and the ones it mixes (as bit masks), for the
// commutation test of the lookahead planner: two gates commute when every
// qubit they share is a block (non-mixed) qubit of both -- for each value of
// the shared qubits the two act on disjoint qubits.  Exact for the snapped
// matrices the kernels apply (mixed_bits uses the same structural zeros).
struct GateQubits {
  uint64_t all = 0, mix = 0;
};
static GateQubits gate_qubits(const LaunchStructure& ls) {
  GateQubits q;
  for (int t : ls.sub_targets) q.all |= uint64_t{1} << t;
  for (int c : ls.controls) q.all |= uint64_t{1} << c;
  if (ls.klass != KernelClass::Diagonal && ls.klass != KernelClass::Identity)
    for (int b : mixed_bits(ls)) q.mix |= uint64_t{1} << ls.sub_targets[b];
  return q;
}

static std::vector<PassStep> plan_passes_window(const std::vector<LaunchStructure>& gates, int n,
                                                const PassConfig& cfg, int window) {
  std::vector<PassStep> steps;
  const int L = cfg.run_log2, M = cfg.tile_log2;
  const int hmax = M - L;
  const bool passes_possible = n >= M;
  const int run_table = 8 << hmax;
  const int G = static_cast<int>(gates.size());

  // per gate: pass role, mixed qubits at or above L, blob bytes, qubit masks
  std::vector<PassRole> role(G, PassRole::Standalone);
  std::vector<std::vector<int>> mixed_hi(G);
  std::vector<int> bytes(G, 0);
  std::vector<GateQubits> qb(G);
  std::vector<char> perm(G, 0);  // in a run of >= min_permute_run consecutive qubit permutations
  for (int i = 0; i < G; ++i) {
    const LaunchStructure& ls = gates[i];
    if (ls.klass == KernelClass::Identity) continue;
    qb[i] = gate_qubits(ls);
    perm[i] = passes_possible && cfg.min_permute_run > 0 && qubit_permutation(ls, nullptr);
    PassRole r = passes_possible ? pass_role(ls, cfg) : PassRole::Standalone;
    if (r != PassRole::Standalone && !cfg.force && pass_op_sweeps(ls, cfg) >= standalone_sweeps(ls, cfg))
      r = PassRole::Standalone;  // cheaper on its own kernel
    role[i] = r;
    if (r == PassRole::Gen)
      for (int b : mixed_bits(ls))
        if (ls.sub_targets[b] >= L) mixed_hi[i].push_back(ls.sub_targets[b]);
    bytes[i] = r == PassRole::Standalone ? 0 : pass_op_bytes(ls, cfg);
  }
  for (int i = 0; i < G;) {  // keep only the permutations inside long enough runs (identities ignored)
    if (!perm[i]) {
      ++i;
      continue;
    }
    std::vector<int> run;
    int j = i;
    for (; j < G; ++j) {
      if (gates[j].klass == KernelClass::Identity) continue;
      if (!perm[j]) break;
      run.push_back(j);
    }
    if (static_cast<int>(run.size()) < cfg.min_permute_run)
      for (int g : run) perm[g] = 0;
    i = j;
  }

  auto emit_standalone = [&](int g) {
    PassStep s;
    s.gates.push_back(g);
    steps.push_back(std::move(s));
  };
  // a finished pass: kept when it beats launching its gates one by one
  auto emit_pass = [&](const std::vector<int>& cur, const std::vector<int>& cur_high) {
    double alone = 0.0, inside = cfg.base_sweeps;
    for (int g : cur) {
      alone += standalone_sweeps(gates[g], cfg);
      inside += pass_op_sweeps(gates[g], cfg);
    }
    if (cfg.force || (cur.size() >= 2 && inside < alone)) {
      PassStep s;
      s.is_pass = true;
      s.gates = cur;
      s.high = cur_high;
      // pad with the lowest free qubits above the runs (fills the tile)
      for (int q = L; q < n && static_cast<int>(s.high.size()) < hmax; ++q)
        if (std::find(s.high.begin(), s.high.end(), q) == s.high.end()) s.high.push_back(q);
      std::sort(s.high.begin(), s.high.end());
      steps.push_back(std::move(s));
    } else {
      for (int g : cur) emit_standalone(g);
    }
  };

  // Lookahead (commutation-aware) grouping: a pass opened at the first
  // remaining gate takes later gates that fit it AND commute with every gate
  // passed over so far (those keep their order and come later); gates that
  // do not fit, standalone gates and permutations are passed over.  Gates of
  // a pass keep program order among themselves.  window 0: the in-order
  // greedy planner (a pass ends at the first gate it cannot take).
  std::vector<char> done(G, 0);
  for (int i = 0; i < G; ++i) done[i] = gates[i].klass == KernelClass::Identity;
  int head = 0;
  while (true) {
    while (head < G && done[head]) ++head;
    if (head >= G) break;
    const int i = head;
    if (perm[i]) {
      // a run of consecutive qubit permutations (identity gates in between ignored)
      std::vector<int> run;
      int j = i;
      for (; j < G; ++j) {
        if (done[j]) continue;
        if (!perm[j]) break;
        run.push_back(j);
      }
      PassStep s;
      s.is_permute = true;
      s.gates = run;
      for (int g : run) done[g] = 1;
      steps.push_back(std::move(s));
      continue;
    }
    if (role[i] == PassRole::Standalone) {
      emit_standalone(i);
      done[i] = 1;
      continue;
    }
    std::vector<int> cur{i};
    std::vector<int> cur_high = mixed_hi[i];
    int cur_bytes = run_table + 4 * 1024 + bytes[i];  // room for a few LAYOUT records + per-thread tables
    done[i] = 1;
    uint64_t skip_all = 0, skip_mix = 0;  // qubits of the gates passed over / the qubits they mix
    int scanned = 0;
    for (int j = i + 1; j < G && scanned < (window > 0 ? window : 1 << 30); ++j) {
      if (done[j]) continue;
      ++scanned;
      bool take = role[j] != PassRole::Standalone && !perm[j] && (qb[j].all & skip_mix) == 0 &&
                  (qb[j].mix & skip_all) == 0;
      std::vector<int> need;
      if (take) {
        need = cur_high;
        for (int q : mixed_hi[j])
          if (std::find(need.begin(), need.end(), q) == need.end()) need.push_back(q);
        // ops + RUN headers must stay within kPassMaxOps (128): at most 2 records per gate
        take = static_cast<int>(need.size()) <= hmax && 2 * (static_cast<int>(cur.size()) + 1) <= 128 &&
               static_cast<int>(cur.size()) < cfg.max_ops && cur_bytes + bytes[j] <= cfg.max_blob;
      }
      if (take) {
        cur.push_back(j);
        cur_high = need;
        cur_bytes += bytes[j];
        done[j] = 1;
      } else {
        if (window == 0) break;  // in-order greedy: the pass ends at the first gate it cannot take
        skip_all |= qb[j].all;
        skip_mix |= qb[j].mix;
        if (skip_mix == (n >= 64 ? ~uint64_t{0} : (uint64_t{1} << n) - 1)) break;  // nothing can commute past
      }
    }
    emit_pass(cur, cur_high);
  }
  return steps;
}

// Estimated sweeps of a plan with the planner's own cost model.
static double plan_sweeps(const std::vector<PassStep>& steps, const std::vector<LaunchStructure>& gates,
                          const PassConfig& cfg) {
  double t = 0.0;
  for (const PassStep& s : steps) {
    if (s.is_permute) {
      t += 1.0;
    } else if (s.is_pass) {
      t += cfg.base_sweeps;
      for (int g : s.gates) t += pass_op_sweeps(gates[g], cfg);
    } else {
      t += standalone_sweeps(gates[s.gates.front()], cfg);
    }
  }
  return t;
}

// Both planners; the lookahead plan is taken when the cost model says it
// saves at least a third of a sweep (B200: RQC-30 k <= 2 57 -> 35 sweeps,
// 551 -> 452 ms; QAOA-30 c64 k = 1 71 -> 31, 310 -> 243 ms), else the
// in-order plan -- on equal sweep counts the hoisted gates made QFT-30's
// passes ~3% slower (profiles/r02/planner_ab.txt).  TSG_PASS_LOOKAHEAD=<window>
// sets the window (default 256; 0: in-order only).
std::vector<PassStep> plan_passes(const std::vector<LaunchStructure>& gates, int n, const PassConfig& cfg) {
  static const int window = [] {
    const char* e = std::getenv("TSG_PASS_LOOKAHEAD");
    return e ? std::max(0, std::atoi(e)) : 256;
  }();
  std::vector<PassStep> in_order = plan_passes_window(gates, n, cfg, 0);
  if (window == 0 || cfg.force) return in_order;
  std::vector<PassStep> ahead = plan_passes_window(gates, n, cfg, window);
  return plan_sweeps(ahead, gates, cfg) + 0.34 <= plan_sweeps(in_order, gates, cfg) ? ahead : in_order;
}

}  // namespace tilesim
