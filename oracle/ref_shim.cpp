// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the reference's own gatecore + circuit sources
// (/root/reference/proj/src/{complex_matrix,gate,circuit}.cpp, compiled
// unmodified by oracle/Makefile into oracle/_ref/libtsref.so).  Used to pin
// the restatement in oracle/oracle.cpp and to generate tests/golden/.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "tilesim/circuit.hpp"
#include "tilesim/complex_matrix.hpp"
#include "tilesim/errors.hpp"
#include "tilesim/gate.hpp"
#include "tilesim/prng.hpp"

using namespace tilesim;

static thread_local std::string g_err;

static void put_matrix(const GateMatrix& m, double* out) {
  const auto& e = m.entries();
  for (size_t i = 0; i < e.size(); ++i) {
    out[2 * i] = e[i].real();
    out[2 * i + 1] = e[i].imag();
  }
}
static GateMatrix get_matrix(int k, const double* m) {
  GateMatrix g(k);
  auto& e = g.entries();
  for (size_t i = 0; i < e.size(); ++i) e[i] = cplx{m[2 * i], m[2 * i + 1]};
  return g;
}

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// make_named_gate (circuit.cpp:135): sorted targets + permuted matrix
int ref_named_gate(const char* name, const double* p, int np, const int* q, int nq, int* k, int* t, double* m) {
  try {
    Gate g = make_named_gate(name, std::vector<double>(p, p + np), std::vector<int>(q, q + nq));
    *k = g.k();
    for (int i = 0; i < g.k(); ++i) t[i] = g.targets[i];
    put_matrix(g.matrix, m);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

int ref_random_unitary(int k, uint64_t seed, int skip, double* out) {
  Prng rng(seed);
  for (int i = 0; i < skip; ++i) random_unitary(k, rng);
  put_matrix(random_unitary(k, rng), out);
  return 0;
}

void ref_prng_stream(uint64_t seed, int count, uint64_t* u, double* normals) {
  Prng a(seed), b(seed);
  for (int i = 0; i < count; ++i) u[i] = a.next_u64();
  for (int i = 0; i < count; ++i) normals[i] = b.normal();
}

int ref_classify(double x, double zt, double ot) { return (int)classify_scalar(x, zt, ot); }

int ref_profile(int k, const double* m, double zt, double ot, uint8_t* kinds, uint64_t* counts) {
  SparsityProfile p = sparsity_profile(get_matrix(k, m), zt, ot);
  for (size_t i = 0; i < p.kinds.size(); ++i) {
    kinds[2 * i] = (uint8_t)p.kinds[i].re;
    kinds[2 * i + 1] = (uint8_t)p.kinds[i].im;
  }
  counts[0] = p.n_general;
  counts[1] = p.n_one;
  counts[2] = p.n_minus_one;
  counts[3] = p.op_count;
  return 0;
}

int ref_is_unitary(int k, const double* m, double tol) { return is_unitary(get_matrix(k, m), tol) ? 1 : 0; }

int ref_fuse(int k1, const int* t1, const double* m1, int k2, const int* t2, const double* m2, int* ok, int* ot,
             double* om) {
  try {
    Gate a = make_gate(get_matrix(k1, m1), std::vector<int>(t1, t1 + k1));
    Gate b = make_gate(get_matrix(k2, m2), std::vector<int>(t2, t2 + k2));
    Gate f = fuse_matrices(a, b);
    *ok = f.k();
    for (int i = 0; i < f.k(); ++i) ot[i] = f.targets[i];
    put_matrix(f.matrix, om);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

int ref_expand(int k, const int* t, const double* m, int ku, const int* tu, double* out) {
  try {
    Gate g = make_gate(get_matrix(k, m), std::vector<int>(t, t + k));
    put_matrix(expand_gate(g, std::vector<int>(tu, tu + ku)), out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

int ref_make_gate_arg_order(int k, const int* q, const double* m, int* t, double* out) {
  try {
    Gate g = make_gate_arg_order(get_matrix(k, m), std::vector<int>(q, q + k));
    for (int i = 0; i < k; ++i) t[i] = g.targets[i];
    put_matrix(g.matrix, out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// parse_circuit (circuit.cpp:225): returns gate count or -1 (error text via
// ref_last_error, with line/column as the reference formats it)
int ref_parse_count(const char* text, int* n_qubits) {
  try {
    Circuit c = parse_circuit(text);
    *n_qubits = c.n_qubits;
    return (int)c.gates.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
