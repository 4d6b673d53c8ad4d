// tilesim/sim.hpp -- SPEC's kernel + sim module as C++ for
// host code written against the reference, implemented header-only over the
// C ABI (tilesim_cuda.h) of the B200 library.  Names and meaning follow SPEC:
//
//   init_zero_state(n, precision)
//   plan_kernel(g, n, s, zero_tol, one_tol,
//               runtime_matrix)
//   apply_kernel(plan, sv, override, t_b, t_e)
//   run_circuit(c, sv, tolerances)
//   norm(sv), compare_states(a, b)
//
// Errors come back as the reference's exception types (tilesim/errors.hpp):
// class 1 -> ParseError, 2 -> ConfigError, 3 -> SimError.  The state lives in
// B200 HBM; there is no CPU path behind these calls.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "tilesim/circuit.hpp"
#include "tilesim/errors.hpp"
#include "tilesim_cuda.h"

namespace tilesim {

enum class Precision { F32 = 32, F64 = 64 };

inline void check_tsg(int rc) {
  if (rc == TSG_OK) return;
  const std::string msg = tsg_last_error();
  if (rc == TSG_ERR_PARSE) throw ParseError(msg);
  if (rc == TSG_ERR_CONFIG) throw ConfigError(msg);
  throw SimError(msg);
}

namespace detail {
inline tsg_ctx* default_ctx() {
  static std::unique_ptr<tsg_ctx, int (*)(tsg_ctx*)> ctx{[] {
                                                           tsg_ctx* c = nullptr;
                                                           check_tsg(tsg_ctx_create(0, &c));
                                                           return c;
                                                         }(),
                                                         tsg_ctx_destroy};
  return ctx.get();
}

inline std::vector<double> interleaved(const GateMatrix& m) {
  std::vector<double> out;
  out.reserve(2 * m.entries().size());
  for (const cplx& v : m.entries()) {
    out.push_back(v.real());
    out.push_back(v.imag());
  }
  return out;
}

// a C-ABI circuit handle holding the same gates (sorted targets, same bits)
inline std::unique_ptr<tsc_circuit, int (*)(tsc_circuit*)> to_handle(const Circuit& c) {
  tsc_circuit* h = nullptr;
  check_tsg(tsc_circuit_create(c.n_qubits, &h));
  std::unique_ptr<tsc_circuit, int (*)(tsc_circuit*)> out{h, tsc_circuit_destroy};
  for (const Gate& g : c.gates) {
    const std::vector<double> m = interleaved(g.matrix);
    check_tsg(tsc_circuit_add_matrix(h, g.k(), g.targets.data(), m.data()));
  }
  return out;
}
}  // namespace detail

// Statevector: SoA re/im in HBM, f64 or f32.
class Statevector {
 public:
  Statevector(int n, Precision p) : n_(n), p_(p) {
    tsg_state* s = nullptr;
    check_tsg(tsg_state_create(detail::default_ctx(), n, static_cast<int>(p), &s));
    st_.reset(s);
  }
  int n() const { return n_; }
  Precision precision() const { return p_; }
  tsg_state* handle() const { return st_.get(); }
  uint64_t size() const { return uint64_t{1} << n_; }

  void init_zero() { check_tsg(tsg_state_init_zero(handle())); }
  void init_basis(uint64_t x) { check_tsg(tsg_state_init_basis(handle(), x)); }
  void upload(const std::vector<double>& re, const std::vector<double>& im) {
    if (re.size() != size() || im.size() != size()) throw ConfigError("host arrays must have 2^n entries");
    check_tsg(tsg_state_upload(handle(), re.data(), im.data()));
  }
  std::pair<std::vector<double>, std::vector<double>> download(uint64_t begin = 0, uint64_t count = ~uint64_t{0}) const {
    if (count == ~uint64_t{0}) count = size() - begin;
    std::vector<double> re(count), im(count);
    check_tsg(tsg_state_download_range(handle(), begin, count, re.data(), im.data()));
    return {std::move(re), std::move(im)};
  }

 private:
  int n_;
  Precision p_;
  std::unique_ptr<tsg_state, int (*)(tsg_state*)> st_{nullptr, tsg_state_destroy};
};

inline Statevector init_zero_state(int n, Precision p) {
  Statevector sv(n, p);
  sv.init_zero();
  return sv;
}

// KernelPlan: an immutable device plan of one gate.
class KernelPlan {
 public:
  KernelPlan(const Gate& g, int n, double zero_tol, double one_tol, bool runtime_matrix) : k_(g.k()) {
    const std::vector<double> m = detail::interleaved(g.matrix);
    tsg_plan* p = nullptr;
    check_tsg(tsg_plan_create(detail::default_ctx(), n, g.k(), g.targets.data(), m.data(), zero_tol, one_tol,
                              runtime_matrix ? 1 : 0, &p));
    plan_.reset(p);
  }
  int k() const { return k_; }
  tsg_plan* handle() const { return plan_.get(); }
  tsg_plan_info info() const {
    tsg_plan_info i{};
    check_tsg(tsg_plan_info_get(handle(), &i));
    return i;
  }

 private:
  int k_;
  std::unique_ptr<tsg_plan, int (*)(tsg_plan*)> plan_{nullptr, tsg_plan_destroy};
};

// s (SPEC's lower-region lane count) is a CPU-vectorisation parameter; the
// B200 kernels pick their own layout, so only s = 0 group indexing is exposed
// for t ranges (the GPU kernel ABI).
inline KernelPlan plan_kernel(const Gate& g, int n, int s = 0, double zero_tol = 1e-8, double one_tol = 1e-8,
                              bool runtime_matrix = false) {
  if (s != 0) throw ConfigError("plan_kernel: the B200 build plans with s = 0 (t over [0, 2^(n-k)))");
  return KernelPlan(g, n, zero_tol, one_tol, runtime_matrix);
}

inline void apply_kernel(const KernelPlan& plan, Statevector& sv, const GateMatrix* matrix_override = nullptr,
                         uint64_t t_begin = 0, uint64_t t_end = ~uint64_t{0}) {
  std::vector<double> ov;
  if (matrix_override) ov = detail::interleaved(*matrix_override);
  check_tsg(tsg_apply(sv.handle(), plan.handle(), matrix_override ? ov.data() : nullptr, t_begin, t_end));
}

struct RunReport {
  double planning_s = 0, execution_s = 0;
  uint64_t gates = 0, launches = 0, total_op_count = 0;
};

// run_circuit: plan every gate once, apply in order on the GPU.
inline RunReport run_circuit(const Circuit& c, Statevector& sv, double zero_tol = 1e-8, double one_tol = 1e-8) {
  if (c.n_qubits != sv.n()) throw ConfigError("run_circuit: circuit and statevector qubit counts differ");
  auto h = detail::to_handle(c);
  tsg_program* p = nullptr;
  check_tsg(tsg_program_create(detail::default_ctx(), h.get(), zero_tol, one_tol, static_cast<int>(sv.precision()), &p));
  std::unique_ptr<tsg_program, int (*)(tsg_program*)> prog{p, tsg_program_destroy};
  tsg_run_report r{};
  check_tsg(tsg_program_run(sv.handle(), p, 0, &r));
  return RunReport{r.planning_s, r.execution_s, r.gates, r.launches, r.total_op_count};
}

inline double norm(const Statevector& sv) {
  double out = 0;
  check_tsg(tsg_norm(sv.handle(), &out));
  return out;
}

inline double compare_states(const Statevector& a, const Statevector& b) {
  double out = 0;
  check_tsg(tsg_compare_states(a.handle(), b.handle(), &out));
  return out;
}

}  // namespace tilesim
