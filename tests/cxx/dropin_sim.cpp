// SPEC's sim/kernel module names (tilesim/sim.hpp) driven from C++:
// init_zero_state, plan_kernel/apply_kernel with t sub-ranges, run_circuit,
// norm, compare_states -- on the B200 through the C ABI.
//   dropin_sim         -> host-only checks (compiles, links, error mapping)
//   dropin_sim --gpu   -> device checks (SPEC.md:466 X example, partition
//                         equivalence, HES-12 unitarity SPEC.md:548)
#include <cmath>
#include <cstdio>
#include <cstring>

#include "tilesim/circuit.hpp"
#include "tilesim/errors.hpp"
#include "tilesim/sim.hpp"

using namespace tilesim;

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  try {
    plan_kernel(make_named_gate("x", {}, {1}), 2, 1);
    std::fprintf(stderr, "s != 0 accepted\n");
    return 1;
  } catch (const ConfigError&) {
  }
  if (!gpu) {
    std::printf("host checks ok\n");
    return 0;
  }
  // X on qubit 1: |01> -> |11>
  Statevector sv = init_zero_state(2, Precision::F64);
  sv.init_basis(1);
  apply_kernel(plan_kernel(make_named_gate("x", {}, {1}), 2), sv);
  auto [re, im] = sv.download();
  if (re[3] != 1.0 || re[1] != 0.0) return std::fprintf(stderr, "X example failed\n"), 1;

  // disjoint t ranges compose to the full application
  Prng rng(7);
  const Gate g = make_gate(random_unitary(3, rng), {1, 4, 9});
  Statevector a(12, Precision::F64), b(12, Precision::F64);
  a.init_basis(77);
  b.init_basis(77);
  KernelPlan p = plan_kernel(g, 12);
  apply_kernel(p, a);
  const uint64_t T = uint64_t{1} << (12 - 3);
  apply_kernel(p, b, nullptr, 0, T / 3);
  apply_kernel(p, b, nullptr, T / 3, T);
  const double part = compare_states(a, b);

  // HES-12, 10 Trotter steps: norm 1 within 1e-10
  Statevector h = init_zero_state(12, Precision::F64);
  RunReport rep = run_circuit(gen_benchmark(BenchmarkKind::HES, 12, 10, 1), h);
  const double nrm = norm(h);
  std::printf("partition maxdiff %.3e, HES-12 norm-1 %.3e, %llu gates\n", part, nrm - 1.0,
              static_cast<unsigned long long>(rep.gates));
  return (part <= 1e-13 && std::fabs(nrm - 1.0) <= 1e-10) ? 0 : 1;
}
