// gatecore of the B200 build: PRNG, scalar classification, unitary checks,
// random unitaries, gate construction and the fusion product.
// Reference semantics: proj/src/complex_matrix.cpp, proj/src/gate.cpp,
// proj/include/tilesim/prng.hpp.  Compiled with -ffp-contract=off so that the
// complex products below round exactly like the reference's.
#include <algorithm>
#include <iterator>

#include "tilesim/core.hpp"

namespace tilesim {

// ------------------------------------------------------------------ errors
static std::string with_location(const std::string& what, int line, int column) {
  if (line <= 0) return what;
  std::string s = "line " + std::to_string(line);
  if (column > 0) s += ", column " + std::to_string(column);
  return s + ": " + what;
}

ParseError::ParseError(const std::string& what, int line, int column)
    : std::runtime_error(with_location(what, line, column)), line_(line), column_(column) {}

// -------------------------------------------------------------------- prng
namespace {
inline uint64_t splitmix(uint64_t& x) {
  uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline uint64_t rol(uint64_t v, int r) { return (v << r) | (v >> (64 - r)); }

// Complex product rounded as g++ lowers std::complex<double>::operator*
// without FMA contraction: (ac - bd) + (ad + bc)i.
inline cplx mul(const cplx& x, const cplx& y) {
  const double a = x.real(), b = x.imag(), c = y.real(), d = y.imag();
  return {a * c - b * d, a * d + b * c};
}
}  // namespace

Prng::Prng(uint64_t seed) {
  uint64_t x = seed;
  for (uint64_t& w : st_) w = splitmix(x);
}

uint64_t Prng::next_u64() {
  const uint64_t out = rol(st_[1] * 5, 7) * 9;
  const uint64_t sh = st_[1] << 17;
  st_[2] ^= st_[0];
  st_[3] ^= st_[1];
  st_[1] ^= st_[2];
  st_[0] ^= st_[3];
  st_[2] ^= sh;
  st_[3] = rol(st_[3], 45);
  return out;
}

double Prng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

double Prng::normal() {
  if (has_cached_) {
    has_cached_ = false;
    return cached_;
  }
  double u1 = uniform();
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  const double u2 = uniform();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 6.283185307179586476925286766559 * u2;
  cached_ = radius * std::sin(angle);
  has_cached_ = true;
  return radius * std::cos(angle);
}

Prng Prng::split() {
  uint64_t x = next_u64();
  return Prng(splitmix(x));
}

// ----------------------------------------------------------- classification
const char* to_string(ScalarKind kind) {
  static const char* names[] = {"zero", "one", "minus_one", "general"};
  const auto i = static_cast<unsigned>(kind);
  return i < 4 ? names[i] : "?";
}

GateMatrix GateMatrix::identity(int k) {
  GateMatrix m(k);
  for (uint64_t i = 0; i < m.dim(); ++i) m.at(i, i) = 1.0;
  return m;
}

bool GateMatrix::finite() const {
  return std::all_of(e_.begin(), e_.end(),
                     [](const cplx& v) { return std::isfinite(v.real()) && std::isfinite(v.imag()); });
}

bool is_unitary(const GateMatrix& m, double tol) {
  if (!m.finite()) return false;
  const uint64_t d = m.dim();
  for (uint64_t r = 0; r < d; ++r) {
    for (uint64_t c = 0; c < d; ++c) {
      cplx dot(0.0, 0.0);
      for (uint64_t j = 0; j < d; ++j) dot += mul(m.at(r, j), std::conj(m.at(c, j)));
      if (std::abs(dot - cplx(r == c ? 1.0 : 0.0, 0.0)) > tol) return false;
    }
  }
  return true;
}

uint64_t op_count(const SparsityProfile& p) { return 2 * p.n_general + p.n_one + p.n_minus_one; }

SparsityProfile sparsity_profile(const GateMatrix& m, double zero_tol, double one_tol) {
  SparsityProfile p;
  p.kinds.resize(m.entries().size());
  uint64_t count[4] = {0, 0, 0, 0};
  for (size_t i = 0; i < m.entries().size(); ++i) {
    const ScalarKind kr = classify_scalar(m.entries()[i].real(), zero_tol, one_tol);
    const ScalarKind ki = classify_scalar(m.entries()[i].imag(), zero_tol, one_tol);
    p.kinds[i] = {kr, ki};
    ++count[static_cast<int>(kr)];
    ++count[static_cast<int>(ki)];
  }
  p.n_one = count[1];
  p.n_minus_one = count[2];
  p.n_general = count[3];
  p.op_count = op_count(p);
  return p;
}

GateMatrix random_unitary(int k, Prng& rng) {
  GateMatrix m(k);
  for (cplx& v : m.entries()) {
    const double re = rng.normal();
    const double im = rng.normal();
    v = cplx(re, im);
  }
  const uint64_t d = m.dim();
  for (uint64_t col = 0; col < d; ++col) {
    for (uint64_t prev = 0; prev < col; ++prev) {  // modified Gram-Schmidt
      cplx proj(0.0, 0.0);
      for (uint64_t r = 0; r < d; ++r) proj += mul(std::conj(m.at(r, prev)), m.at(r, col));
      for (uint64_t r = 0; r < d; ++r) m.at(r, col) -= mul(proj, m.at(r, prev));
    }
    double sq = 0.0;
    for (uint64_t r = 0; r < d; ++r) sq += m.at(r, col).real() * m.at(r, col).real() + m.at(r, col).imag() * m.at(r, col).imag();
    const double scale = 1.0 / std::sqrt(sq);
    for (uint64_t r = 0; r < d; ++r) m.at(r, col) = cplx(m.at(r, col).real() * scale, m.at(r, col).imag() * scale);
  }
  return m;
}

// ------------------------------------------------------------------- gates
namespace {
// bit b of `v` lands at position pos[b]
inline uint64_t deposit(uint64_t v, const int* pos, int count) {
  uint64_t out = 0;
  for (int b = 0; b < count; ++b) out |= ((v >> b) & 1u) << pos[b];
  return out;
}
// inverse: collect the bits at pos[] into the low bits
inline uint64_t extract(uint64_t v, const int* pos, int count) {
  uint64_t out = 0;
  for (int b = 0; b < count; ++b) out |= ((v >> pos[b]) & 1u) << b;
  return out;
}
std::vector<int> locate(const std::vector<int>& sub, const std::vector<int>& super) {
  std::vector<int> at;
  at.reserve(sub.size());
  for (int q : sub) {
    const auto it = std::lower_bound(super.begin(), super.end(), q);
    if (it == super.end() || *it != q) throw std::invalid_argument("gate targets not contained in union set");
    at.push_back(static_cast<int>(it - super.begin()));
  }
  return at;
}
}  // namespace

Gate make_gate(GateMatrix matrix, std::vector<int> targets, std::string name, std::vector<double> params) {
  if (targets.empty()) throw std::invalid_argument("gate needs at least one target qubit");
  if (std::adjacent_find(targets.begin(), targets.end(), [](int a, int b) { return a >= b; }) != targets.end())
    throw std::invalid_argument("gate targets must be strictly increasing");
  if (targets.front() < 0) throw std::invalid_argument("negative target qubit");
  if (matrix.k() != static_cast<int>(targets.size()))
    throw std::invalid_argument("matrix size does not match target count");
  if (!matrix.finite()) throw std::invalid_argument("gate matrix has non-finite entries");
  Gate g;
  g.matrix = std::move(matrix);
  g.targets = std::move(targets);
  g.name = std::move(name);
  g.params = std::move(params);
  return g;
}

Gate make_gate_arg_order(const GateMatrix& m, const std::vector<int>& arg_qubits, std::string name,
                         std::vector<double> params) {
  const int k = static_cast<int>(arg_qubits.size());
  if (m.k() != k) throw std::invalid_argument("matrix size does not match argument count");
  std::vector<int> sorted(arg_qubits);
  std::sort(sorted.begin(), sorted.end());
  if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
    throw std::invalid_argument("duplicate qubit in gate arguments");
  std::vector<int> dest(k);  // argument j -> bit position in sorted order
  bool identity_perm = true;
  for (int j = 0; j < k; ++j) {
    dest[j] = static_cast<int>(std::lower_bound(sorted.begin(), sorted.end(), arg_qubits[j]) - sorted.begin());
    identity_perm &= dest[j] == j;
  }
  if (identity_perm) return make_gate(m, sorted, std::move(name), std::move(params));
  GateMatrix out(k);
  const uint64_t d = m.dim();
  for (uint64_t r = 0; r < d; ++r) {
    const uint64_t rr = deposit(r, dest.data(), k);
    for (uint64_t c = 0; c < d; ++c) out.at(rr, deposit(c, dest.data(), k)) = m.at(r, c);
  }
  return make_gate(std::move(out), std::move(sorted), std::move(name), std::move(params));
}

std::vector<int> wire_union(const std::vector<int>& a, const std::vector<int>& b) {
  std::vector<int> u;
  u.reserve(a.size() + b.size());
  std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(u));
  return u;
}

GateMatrix expand_gate(const Gate& g, const std::vector<int>& union_targets) {
  const int m = static_cast<int>(union_targets.size());
  const std::vector<int> own = locate(g.targets, union_targets);
  std::vector<int> other;
  for (int b = 0; b < m; ++b)
    if (std::find(own.begin(), own.end(), b) == own.end()) other.push_back(b);
  GateMatrix out(m);
  const uint64_t dim = out.dim();
  // every union index decomposes into (own bits, other bits); the embedded
  // operator is g on the own bits and identity on the rest.
  for (uint64_t r = 0; r < dim; ++r) {
    const uint64_t gr = extract(r, own.data(), g.k());
    const uint64_t rest = r & ~deposit(~uint64_t{0}, own.data(), g.k());
    for (uint64_t gc = 0; gc < g.matrix.dim(); ++gc) out.at(r, rest | deposit(gc, own.data(), g.k())) = g.matrix.at(gr, gc);
  }
  return out;
}

Gate fuse_matrices(const Gate& first, const Gate& second, int hard_cap) {
  std::vector<int> wires = wire_union(first.targets, second.targets);
  const int m = static_cast<int>(wires.size());
  if (m > hard_cap)
    throw std::invalid_argument("fused gate would span " + std::to_string(m) + " qubits, above the cap of " +
                                std::to_string(hard_cap));
  const std::vector<int> fpos = locate(first.targets, wires);
  const std::vector<int> spos = locate(second.targets, wires);
  const int kf = first.k(), ks = second.k();

  // Split the second gate's bits into shared (also in first) and second-only,
  // and the first gate's bits into shared and first-only.  For a union row r
  // and column c the product entry is
  //   sum_w S[ row_s(r) ][ cs(c) | w_s ] * F[ rf(r) | w_f ][ col_f(c) ]
  // over shared assignments w in ascending order.
  std::vector<int> sh_in_f, sh_in_s;  // shared bit positions local to F / S
  uint64_t s_only_local = 0, f_only_local = 0;  // local-bit masks
  for (int b = 0; b < m; ++b) {
    const auto fi = std::find(fpos.begin(), fpos.end(), b);
    const auto si = std::find(spos.begin(), spos.end(), b);
    const bool in_f = fi != fpos.end(), in_s = si != spos.end();
    if (in_f && in_s) {
      sh_in_f.push_back(static_cast<int>(fi - fpos.begin()));
      sh_in_s.push_back(static_cast<int>(si - spos.begin()));
    } else if (in_f) {
      f_only_local |= uint64_t{1} << (fi - fpos.begin());
    } else {
      s_only_local |= uint64_t{1} << (si - spos.begin());
    }
  }
  const int nsh = static_cast<int>(sh_in_f.size());
  const uint64_t dim = uint64_t{1} << m, nw = uint64_t{1} << nsh;
  std::vector<uint64_t> wf(nw), ws(nw);
  for (uint64_t w = 0; w < nw; ++w) {
    wf[w] = deposit(w, sh_in_f.data(), nsh);
    ws[w] = deposit(w, sh_in_s.data(), nsh);
  }
  GateMatrix out(m);
  const GateMatrix& F = first.matrix;
  const GateMatrix& S = second.matrix;
  // per-row / per-column local indices once (the product loop below keeps
  // the reference's accumulation order: w ascending, real and imaginary
  // sums separately -- bit-exact)
  const uint64_t dF = F.dim(), dS = S.dim();
  // (fused blocks are small: stack tables up to 6 qubits)
  uint64_t tab_small[4 * 64];
  std::vector<uint64_t> tab_big(dim > 64 ? 4 * dim : 0);
  uint64_t* const tab = dim > 64 ? tab_big.data() : tab_small;
  uint64_t *srow = tab, *frow = tab + dim, *fcol = tab + 2 * dim, *scol = tab + 3 * dim;
  for (uint64_t x = 0; x < dim; ++x) {
    srow[x] = extract(x, spos.data(), ks) * dS;
    frow[x] = extract(x, fpos.data(), kf) & f_only_local;
    fcol[x] = extract(x, fpos.data(), kf);
    scol[x] = extract(x, spos.data(), ks) & s_only_local;
  }
  for (uint64_t w = 0; w < nw; ++w) wf[w] *= dF;  // row offsets in F
  const cplx* fe = &F.at(0, 0);
  const cplx* se = &S.at(0, 0);
  for (uint64_t r = 0; r < dim; ++r) {
    const cplx* srow_p = se + srow[r];
    const cplx* frow_p = fe + frow[r] * dF;
    for (uint64_t c = 0; c < dim; ++c) {
      const cplx* sp = srow_p + scol[c];
      const cplx* fp = frow_p + fcol[c];
      double acc_re = 0.0, acc_im = 0.0;
      for (uint64_t w = 0; w < nw; ++w) {
        const cplx p = mul(sp[ws[w]], fp[wf[w]]);
        acc_re += p.real();
        acc_im += p.imag();
      }
      out.at(r, c) = cplx(acc_re, acc_im);
    }
  }
  Gate g;
  g.matrix = std::move(out);
  g.targets = std::move(wires);
  return g;
}

}  // namespace tilesim
