// tilesim/core.hpp -- gate algebra of the B200 build ("gatecore").
//
// Same public names and semantics as the reference's gatecore so host code
// written against it drops in:
//   ScalarKind / classify_scalar      proj/include/tilesim/complex_matrix.hpp:16-28
//   GateMatrix                        proj/include/tilesim/complex_matrix.hpp:37-65
//   SparsityProfile / op_count        proj/include/tilesim/complex_matrix.hpp:72-93
//   is_unitary / random_unitary       proj/include/tilesim/complex_matrix.hpp:67,97
//   Gate / make_gate / ...            proj/include/tilesim/gate.hpp:12-48
//   Prng                              proj/include/tilesim/prng.hpp:15-78
//   ParseError / ConfigError / SimError  proj/include/tilesim/errors.hpp:10-47
//
// Arithmetic contract: fuse_matrices, random_unitary and the named-gate table
// produce the same bits as the reference (checked against oracle/_ref and
// tests/golden/).  This translation unit is compiled with -ffp-contract=off.
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace tilesim {

using cplx = std::complex<double>;

// ------------------------------------------------------------------ errors
// Exit-code mapping of SPEC.md:587: ParseError -> 1, ConfigError -> 2,
// SimError -> 3.  ParseError prefixes "line L, column C: " when known.
class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& what, int line = 0, int column = 0);
  int line() const { return line_; }
  int column() const { return column_; }

 private:
  int line_, column_;
};

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct SimError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// -------------------------------------------------------------------- prng
// splitmix64-seeded xoshiro256**, 53-bit uniforms, Box-Muller normals with a
// cached spare.  The algorithm is part of the seed contract.
class Prng {
 public:
  explicit Prng(uint64_t seed);
  uint64_t next_u64();
  double uniform();  // [0, 1)
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint64_t next_below(uint64_t bound) { return next_u64() % bound; }
  double normal();
  Prng split();

 private:
  uint64_t st_[4];
  double cached_ = 0.0;
  bool has_cached_ = false;
};

// ------------------------------------------------------ scalar sparsity
enum class ScalarKind : uint8_t { Zero = 0, One = 1, MinusOne = 2, General = 3 };

inline ScalarKind classify_scalar(double x, double zero_tol, double one_tol) {
  if (std::fabs(x) <= zero_tol) return ScalarKind::Zero;
  if (std::fabs(x - 1.0) <= one_tol) return ScalarKind::One;
  if (std::fabs(x + 1.0) <= one_tol) return ScalarKind::MinusOne;
  return ScalarKind::General;
}
const char* to_string(ScalarKind kind);

// Value a scalar of the given kind is executed as: Zero -> 0, One -> +1,
// MinusOne -> -1, General -> itself.  Kernels run on the snapped matrix, which
// makes "skip zeros, lower +-1 to add/sub" exact by construction.
inline double snap_scalar(double x, ScalarKind k) {
  switch (k) {
    case ScalarKind::Zero: return 0.0;
    case ScalarKind::One: return 1.0;
    case ScalarKind::MinusOne: return -1.0;
    default: return x;
  }
}

// -------------------------------------------------------------- matrices
// Row-major 2^k x 2^k; bit j of a row/column index is the j-th sorted target.
class GateMatrix {
 public:
  GateMatrix() = default;
  explicit GateMatrix(int k) : k_(k), e_(size_t{1} << (2 * k), cplx(0.0, 0.0)) {}
  static GateMatrix identity(int k);

  int k() const { return k_; }
  uint64_t dim() const { return uint64_t{1} << k_; }
  cplx& at(uint64_t r, uint64_t c) { return e_[r * dim() + c]; }
  const cplx& at(uint64_t r, uint64_t c) const { return e_[r * dim() + c]; }
  std::vector<cplx>& entries() { return e_; }
  const std::vector<cplx>& entries() const { return e_; }
  bool finite() const;

 private:
  int k_ = 0;
  std::vector<cplx> e_;
};

bool is_unitary(const GateMatrix& m, double tol);

struct SparsityProfile {
  struct KindPair {
    ScalarKind re, im;
  };
  std::vector<KindPair> kinds;  // row-major, one pair per entry
  uint64_t n_general = 0, n_one = 0, n_minus_one = 0, op_count = 0;
  uint64_t nonzero_scalars() const { return n_general + n_one + n_minus_one; }
};

// 2 per General scalar, 1 per +-1 scalar, 0 per Zero.
uint64_t op_count(const SparsityProfile& p);
SparsityProfile sparsity_profile(const GateMatrix& m, double zero_tol, double one_tol);

// Gaussian complex entries, modified Gram-Schmidt on columns.
GateMatrix random_unitary(int k, Prng& rng);

// ------------------------------------------------------------------ gates
inline constexpr int kFusedQubitCap = 12;

struct Gate {
  GateMatrix matrix;
  std::vector<int> targets;  // strictly increasing
  std::string name;          // empty for raw-matrix / fused gates
  std::vector<double> params;
  int k() const { return static_cast<int>(targets.size()); }
};

// All three throw std::invalid_argument on contract violations, exactly as
// the reference does (gate.cpp:34-93).
Gate make_gate(GateMatrix matrix, std::vector<int> targets, std::string name = {}, std::vector<double> params = {});
Gate make_gate_arg_order(const GateMatrix& m, const std::vector<int>& arg_qubits, std::string name = {},
                         std::vector<double> params = {});
GateMatrix expand_gate(const Gate& g, const std::vector<int>& union_targets);
std::vector<int> wire_union(const std::vector<int>& a, const std::vector<int>& b);

// Gate over the union equal to applying `first` then `second`:
// matrix = expand(second) * expand(first), summed over shared bits only.
Gate fuse_matrices(const Gate& first, const Gate& second, int hard_cap = kFusedQubitCap);

}  // namespace tilesim
