// A translation unit written the way the reference's own sources are: its
// includes are exactly those of proj/src/circuit.cpp:1,10 and gate.cpp:1,
// plus the B200 C ABI.  It uses only reference-surface calls to build a
// circuit (named-gate lowering, the text format, fuse_matrices), then runs it
// on the GPU through tilesim_cuda.h and checks QFT|x> against the closed form
// e^{2 pi i x y / 2^n} / 2^{n/2}.
//
//   dropin_qft            -> build + fuse checks only (host), exit 0
//   dropin_qft --gpu      -> also simulate QFT-12 on the B200 and check it
#include "tilesim/circuit.hpp"

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tilesim/errors.hpp"
#include "tilesim/gate.hpp"
#include "tilesim_cuda.h"

using namespace tilesim;

static int fail(const char* what) {
  std::fprintf(stderr, "dropin_qft: %s (%s)\n", what, tsg_last_error());
  return 1;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  const int n = 12;
  const unsigned x = 0x5A5 & ((1u << n) - 1);
  const double pi = 3.141592653589793238462643383279502884;

  // QFT-n, top-down: h j, cp(pi/2^(j-m)) m j for m < j, swaps
  Circuit c;
  c.n_qubits = n;
  for (int j = n - 1; j >= 0; --j) {
    c.gates.push_back(make_named_gate("h", {}, {j}));
    for (int m = j - 1; m >= 0; --m) c.gates.push_back(make_named_gate("cp", {pi / std::ldexp(1.0, j - m)}, {m, j}));
  }
  for (int i = 0; i < n / 2; ++i) c.gates.push_back(make_named_gate("swap", {}, {i, n - 1 - i}));

  // the text format round-trips the named gates (circuit.hpp:38-40)
  const Circuit back = parse_circuit(serialize_circuit(c));
  if (back.gates.size() != c.gates.size()) return fail("parse(serialize(c)) lost gates");
  try {
    parse_circuit("qubits 2\nfoo 0\n");
    return fail("unknown gate accepted");
  } catch (const ParseError&) {
  }

  // fuse neighbouring gates pairwise up to 3 qubits with the reference's
  // fuse_matrices (gate.hpp:41-44): a left fold, applied in program order
  std::vector<Gate> fused;
  for (const Gate& g : c.gates) {
    if (!fused.empty() && wire_union(fused.back().targets, g.targets).size() <= 3)
      fused.back() = fuse_matrices(fused.back(), g);
    else
      fused.push_back(g);
  }
  std::printf("QFT-%d: %zu gates, %zu after pairwise fusion\n", n, c.gates.size(), fused.size());
  if (!gpu) return 0;

  int devices = 0;
  tsg_device_count(&devices);
  if (devices == 0) return fail("no CUDA device");
  tsg_ctx* ctx = nullptr;
  tsc_circuit* h = nullptr;
  tsg_state* st = nullptr;
  tsg_program* prog = nullptr;
  if (tsg_ctx_create(0, &ctx) || tsc_circuit_create(n, &h)) return fail("context / circuit");
  for (const Gate& g : fused) {
    std::vector<double> m;
    for (const auto& v : g.matrix.entries()) {
      m.push_back(v.real());
      m.push_back(v.imag());
    }
    if (tsc_circuit_add_matrix(h, g.k(), g.targets.data(), m.data())) return fail("add_matrix");
  }
  if (tsg_state_create(ctx, n, 64, &st) || tsg_state_init_basis(st, x)) return fail("state");
  if (tsg_program_create(ctx, h, 1e-8, 1e-8, 64, &prog)) return fail("program");
  tsg_run_report rep{};
  if (tsg_program_run(st, prog, 0, &rep)) return fail("run");
  std::vector<double> re(1u << n), im(1u << n);
  if (tsg_state_download(st, re.data(), im.data())) return fail("download");
  double worst = 0;
  for (unsigned y = 0; y < (1u << n); ++y) {
    const double ph = 2 * pi * static_cast<double>((static_cast<uint64_t>(x) * y) % (1u << n)) / (1u << n);
    const std::complex<double> want = std::polar(std::pow(2.0, -n / 2.0), ph);
    worst = std::max(worst, std::abs(std::complex<double>(re[y], im[y]) - want));
  }
  std::printf("QFT-%d on the GPU: %llu launches, max |dpsi| vs closed form %.3e\n", n,
              static_cast<unsigned long long>(rep.launches), worst);
  tsg_program_destroy(prog);
  tsg_state_destroy(st);
  tsc_circuit_destroy(h);
  tsg_ctx_destroy(ctx);
  return worst <= 1e-10 ? 0 : 1;
}
