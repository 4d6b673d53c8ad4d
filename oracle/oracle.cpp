// =============================================================================
// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY. NOT PART OF THE PRODUCT.
//
// A CPU restatement of the CAST / tilesim algorithm for the hot path
// (applying sparsity-aware fused k-qubit gates to a 2^n statevector) and for
// everything that produces its input (gate algebra, benchmark generators, the
// CircuitTile fusion pass, the cost-model interpolation).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load this library; the product (paper_2503_19894_b200) never links it.
//
// Sources restated (paths relative to /root/reference):
//   gatecore   proj/include/tilesim/{complex_matrix,gate,prng}.hpp,
//              proj/src/{complex_matrix,gate}.cpp
//   circuit    proj/src/circuit.cpp:25-148 (named gate table and matrices)
//   generators SPEC.md:170-178 (+ QAOA, pinned in DESIGN.md §3)
//   tile       SPEC.md:200-304      (Algorithm 1)
//   fusion
//   kernel
//   sim
//
// Parity pinning: the gatecore restatement is checked bit-for-bit against the
// reference's own sources compiled into oracle/_ref (see oracle/Makefile,
// oracle/ref_shim.cpp) and against the committed fixtures in tests/golden/.
// Compile with -ffp-contract=off: the reference is built without -march, so
// its complex products are never contracted into FMAs.
// =============================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using cd = std::complex<double>;
static const double PI = 3.141592653589793238462643383279502884;

// ---------------------------------------------------------------- errors ---
struct Err : std::runtime_error {
  int code;  // 1 parse, 2 config, 3 sim (mirrors SPEC.md:587 exit codes)
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// ------------------------------------------------------------------ prng ---
// xoshiro256** seeded by splitmix64 (proj/include/tilesim/prng.hpp:15-78).
struct Rng {
  uint64_t s[4];
  double spare = 0.0;
  bool have_spare = false;
  static uint64_t sm64(uint64_t* x) {
    *x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) s[i] = sm64(&x);
  }
  static uint64_t rotl(uint64_t v, int r) { return (v << r) | (v >> (64 - r)); }
  uint64_t u64() {
    uint64_t out = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
  }
  double unif() { return (double)(u64() >> 11) * 0x1.0p-53; }
  double unif(double lo, double hi) { return lo + (hi - lo) * unif(); }
  uint64_t below(uint64_t b) { return u64() % b; }
  double gauss() {  // Box-Muller with a cached second value (prng.hpp:43-57)
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double a = unif();
    if (a <= 0.0) a = 0x1.0p-53;
    double b = unif();
    double rad = std::sqrt(-2.0 * std::log(a));
    double ang = 6.283185307179586476925286766559 * b;
    spare = rad * std::sin(ang);
    have_spare = true;
    return rad * std::cos(ang);
  }
};

// -------------------------------------------------------- matrices/gates ---
struct Mat {
  int k = 0;
  std::vector<cd> e;  // row-major 2^k x 2^k
  Mat() {}
  explicit Mat(int kk) : k(kk), e((size_t)1 << (2 * kk), cd(0.0, 0.0)) {}
  size_t dim() const { return (size_t)1 << k; }
  cd& at(size_t r, size_t c) { return e[r * dim() + c]; }
  const cd& at(size_t r, size_t c) const { return e[r * dim() + c]; }
};

struct Gate {
  Mat m;
  std::vector<int> t;  // strictly increasing
  std::string name;
  std::vector<double> p;
};

struct Circ {
  int n = 0;
  std::vector<Gate> g;
};

// complex product written out the way g++ -O3 (no -march) lowers
// std::complex<double>::operator*: re = ac - bd, im = ad + bc.
static inline cd cmul(const cd& x, const cd& y) {
  double a = x.real(), b = x.imag(), c = y.real(), d = y.imag();
  return cd(a * c - b * d, a * d + b * c);
}

// ScalarKind precedence Zero > One > MinusOne > General
// (proj/include/tilesim/complex_matrix.hpp:20-28).
enum : uint8_t { K_ZERO = 0, K_ONE = 1, K_MONE = 2, K_GEN = 3 };
static inline uint8_t kind_of(double x, double zt, double ot) {
  if (std::fabs(x) <= zt) return K_ZERO;
  if (std::fabs(x - 1.0) <= ot) return K_ONE;
  if (std::fabs(x + 1.0) <= ot) return K_MONE;
  return K_GEN;
}

struct Profile {
  std::vector<uint8_t> kre, kim;
  uint64_t gen = 0, one = 0, mone = 0, ops = 0;
};

// proj/src/complex_matrix.cpp:46-76; op_count = 2*General + (One + MinusOne).
static Profile profile_of(const Mat& m, double zt, double ot) {
  Profile p;
  p.kre.resize(m.e.size());
  p.kim.resize(m.e.size());
  for (size_t i = 0; i < m.e.size(); ++i) {
    p.kre[i] = kind_of(m.e[i].real(), zt, ot);
    p.kim[i] = kind_of(m.e[i].imag(), zt, ot);
    for (uint8_t kk : {p.kre[i], p.kim[i]}) {
      if (kk == K_GEN) p.gen++;
      else if (kk == K_ONE) p.one++;
      else if (kk == K_MONE) p.mone++;
    }
  }
  p.ops = 2 * p.gen + p.one + p.mone;
  return p;
}

static bool finite_mat(const Mat& m) {
  for (auto& v : m.e)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
  return true;
}

// proj/src/complex_matrix.cpp:30-44
static bool unitary(const Mat& m, double tol) {
  if (!finite_mat(m)) return false;
  size_t d = m.dim();
  for (size_t r = 0; r < d; ++r)
    for (size_t c = 0; c < d; ++c) {
      cd acc(0.0, 0.0);
      for (size_t j = 0; j < d; ++j) acc += cmul(m.at(r, j), std::conj(m.at(c, j)));
      cd want = (r == c) ? cd(1.0, 0.0) : cd(0.0, 0.0);
      if (std::abs(acc - want) > tol) return false;
    }
  return true;
}

// Gaussian complex entries, then modified Gram-Schmidt over columns
// (proj/src/complex_matrix.cpp:78-101).
static Mat haar_like(int k, Rng& rng) {
  Mat m(k);
  for (auto& v : m.e) {
    double re = rng.gauss();
    double im = rng.gauss();
    v = cd(re, im);
  }
  size_t d = m.dim();
  for (size_t c = 0; c < d; ++c) {
    for (size_t pc = 0; pc < c; ++pc) {
      cd dot(0.0, 0.0);
      for (size_t r = 0; r < d; ++r) dot += cmul(std::conj(m.at(r, pc)), m.at(r, c));
      for (size_t r = 0; r < d; ++r) m.at(r, c) -= cmul(dot, m.at(r, pc));
    }
    double ns = 0.0;
    for (size_t r = 0; r < d; ++r) {
      double x = m.at(r, c).real(), y = m.at(r, c).imag();
      ns += x * x + y * y;
    }
    double inv = 1.0 / std::sqrt(ns);
    for (size_t r = 0; r < d; ++r) m.at(r, c) = cd(m.at(r, c).real() * inv, m.at(r, c).imag() * inv);
  }
  return m;
}

static Gate checked_gate(Mat m, std::vector<int> t, std::string name = "", std::vector<double> p = {}) {
  if (t.empty()) throw Err(2, "gate needs at least one target qubit");
  for (size_t i = 1; i < t.size(); ++i)
    if (t[i - 1] >= t[i]) throw Err(2, "gate targets must be strictly increasing");
  if (t[0] < 0) throw Err(2, "negative target qubit");
  if (m.k != (int)t.size()) throw Err(2, "matrix size does not match target count");
  if (!finite_mat(m)) throw Err(2, "gate matrix has non-finite entries");
  Gate g;
  g.m = std::move(m);
  g.t = std::move(t);
  g.name = std::move(name);
  g.p = std::move(p);
  return g;
}

// Argument-order matrix -> sorted-target gate (proj/src/gate.cpp:52-93):
// index bit j (j-th argument) moves to the rank of that qubit among the sorted.
static Gate gate_from_args(const Mat& m, const std::vector<int>& args, std::string name = "",
                           std::vector<double> p = {}) {
  int k = (int)args.size();
  if (m.k != k) throw Err(2, "matrix size does not match argument count");
  std::vector<int> srt = args;
  std::sort(srt.begin(), srt.end());
  for (int i = 1; i < k; ++i)
    if (srt[i] == srt[i - 1]) throw Err(2, "duplicate qubit in gate arguments");
  std::vector<int> rk(k);
  bool ident = true;
  for (int j = 0; j < k; ++j) {
    rk[j] = (int)(std::lower_bound(srt.begin(), srt.end(), args[j]) - srt.begin());
    ident = ident && rk[j] == j;
  }
  if (ident) return checked_gate(m, srt, name, p);
  size_t d = m.dim();
  std::vector<size_t> mp(d);
  for (size_t i = 0; i < d; ++i) {
    size_t o = 0;
    for (int j = 0; j < k; ++j) o |= ((i >> j) & 1u) << rk[j];
    mp[i] = o;
  }
  Mat q(k);
  for (size_t r = 0; r < d; ++r)
    for (size_t c = 0; c < d; ++c) q.at(mp[r], mp[c]) = m.at(r, c);
  return checked_gate(q, srt, name, p);
}

static std::vector<int> wires_union(const std::vector<int>& a, const std::vector<int>& b) {
  std::vector<int> u;
  std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(u));
  return u;
}

static std::vector<int> index_in(const std::vector<int>& sub, const std::vector<int>& sup) {
  std::vector<int> pos;
  for (int q : sub) {
    auto it = std::lower_bound(sup.begin(), sup.end(), q);
    if (it == sup.end() || *it != q) throw Err(2, "gate targets not contained in union set");
    pos.push_back((int)(it - sup.begin()));
  }
  return pos;
}

static inline size_t scatter_bits(size_t v, const std::vector<int>& pos) {
  size_t o = 0;
  for (size_t j = 0; j < pos.size(); ++j) o |= ((v >> j) & 1u) << pos[j];
  return o;
}

// Embed g into the space of `uni` (proj/src/gate.cpp:95-122).
static Mat embed(const Gate& g, const std::vector<int>& uni) {
  int m = (int)uni.size();
  std::vector<int> pos = index_in(g.t, uni);
  std::vector<int> rest;
  for (int b = 0; b < m; ++b)
    if (std::find(pos.begin(), pos.end(), b) == pos.end()) rest.push_back(b);
  Mat out(m);
  size_t gd = g.m.dim();
  for (size_t x = 0; x < ((size_t)1 << rest.size()); ++x) {
    size_t rb = scatter_bits(x, rest);
    for (size_t r = 0; r < gd; ++r)
      for (size_t c = 0; c < gd; ++c) out.at(rb | scatter_bits(r, pos), rb | scatter_bits(c, pos)) = g.m.at(r, c);
  }
  return out;
}

// fuse(first, second) = embed(second) * embed(first), summing only over the
// bits shared by both gates, in ascending order of the shared assignment,
// from 0+0i (proj/src/gate.cpp:131-220).
static Gate fuse2(const Gate& first, const Gate& second, int cap = 12) {
  std::vector<int> u = wires_union(first.t, second.t);
  int m = (int)u.size();
  if (m > cap) throw Err(2, "fused gate would span " + std::to_string(m) + " qubits, above the cap of " + std::to_string(cap));
  std::vector<int> fpos = index_in(first.t, u), spos = index_in(second.t, u);
  std::vector<int> fbit(m, -1), sbit(m, -1);
  for (size_t j = 0; j < fpos.size(); ++j) fbit[fpos[j]] = (int)j;
  for (size_t j = 0; j < spos.size(); ++j) sbit[spos[j]] = (int)j;
  // classify union bits
  std::vector<int> sh_f, sh_s, fo_u, fo_l, so_u, so_l;
  for (int b = 0; b < m; ++b) {
    if (fbit[b] >= 0 && sbit[b] >= 0) {
      sh_f.push_back(fbit[b]);
      sh_s.push_back(sbit[b]);
    } else if (fbit[b] >= 0) {
      fo_u.push_back(b);
      fo_l.push_back(fbit[b]);
    } else {
      so_u.push_back(b);
      so_l.push_back(sbit[b]);
    }
  }
  size_t d = (size_t)1 << m, nw = (size_t)1 << sh_f.size();
  auto gather = [](size_t i, const std::vector<int>& from, const std::vector<int>& to) {
    size_t o = 0;
    for (size_t j = 0; j < from.size(); ++j) o |= ((i >> from[j]) & 1u) << to[j];
    return o;
  };
  std::vector<int> ident_f(fpos.size()), ident_s(spos.size());
  for (size_t j = 0; j < fpos.size(); ++j) ident_f[j] = (int)j;
  for (size_t j = 0; j < spos.size(); ++j) ident_s[j] = (int)j;
  Mat out(m);
  const Mat& F = first.m;
  const Mat& S = second.m;
  for (size_t r = 0; r < d; ++r) {
    size_t srow = gather(r, spos, ident_s);
    size_t frow_fixed = gather(r, fo_u, fo_l);
    for (size_t c = 0; c < d; ++c) {
      size_t fcol = gather(c, fpos, ident_f);
      size_t scol_fixed = gather(c, so_u, so_l);
      double ar = 0.0, ai = 0.0;
      for (size_t w = 0; w < nw; ++w) {
        cd prod = cmul(S.at(srow, scol_fixed | scatter_bits(w, sh_s)), F.at(frow_fixed | scatter_bits(w, sh_f), fcol));
        ar += prod.real();
        ai += prod.imag();
      }
      out.at(r, c) = cd(ar, ai);
    }
  }
  Gate g;
  g.m = std::move(out);
  g.t = std::move(u);
  return g;
}

// ------------------------------------------------------------ named gates ---
// Gate table and matrices of proj/src/circuit.cpp:25-121 (argument order).
struct NamedInfo {
  const char* nm;
  int arity, params;
};
static const NamedInfo NAMED[] = {{"x", 1, 0},  {"y", 1, 0},   {"z", 1, 0},  {"h", 1, 0},   {"s", 1, 0},   {"sdg", 1, 0},
                                  {"t", 1, 0},  {"tdg", 1, 0}, {"rx", 1, 1}, {"ry", 1, 1},  {"rz", 1, 1},  {"u3", 1, 3},
                                  {"cx", 2, 0}, {"cz", 2, 0},  {"cp", 2, 1}, {"swap", 2, 0}, {"ccx", 3, 0}};

static const NamedInfo* lookup(const std::string& n) {
  for (auto& i : NAMED)
    if (n == i.nm) return &i;
  return nullptr;
}

static Mat m2x2(cd a, cd b, cd c, cd d) {
  Mat m(1);
  m.e = {a, b, c, d};
  return m;
}

static Mat named_argorder(const std::string& nm, const std::vector<double>& p) {
  const double r2 = 0.70710678118654752440084436210485;
  const cd I(0.0, 1.0);
  if (nm == "x") return m2x2(0.0, 1.0, 1.0, 0.0);
  if (nm == "y") return m2x2(0.0, -I, I, 0.0);
  if (nm == "z") return m2x2(1.0, 0.0, 0.0, -1.0);
  if (nm == "h") return m2x2(r2, r2, r2, -r2);
  if (nm == "s") return m2x2(1.0, 0.0, 0.0, I);
  if (nm == "sdg") return m2x2(1.0, 0.0, 0.0, -I);
  if (nm == "t") return m2x2(1.0, 0.0, 0.0, std::polar(1.0, PI / 4.0));
  if (nm == "tdg") return m2x2(1.0, 0.0, 0.0, std::polar(1.0, -PI / 4.0));
  if (nm == "rx") {
    double c = std::cos(p[0] / 2.0), s = std::sin(p[0] / 2.0);
    return m2x2(c, -I * s, -I * s, c);
  }
  if (nm == "ry") {
    double c = std::cos(p[0] / 2.0), s = std::sin(p[0] / 2.0);
    return m2x2(c, -s, s, c);
  }
  if (nm == "rz") return m2x2(std::polar(1.0, -p[0] / 2.0), 0.0, 0.0, std::polar(1.0, p[0] / 2.0));
  if (nm == "u3") {
    double c = std::cos(p[0] / 2.0), s = std::sin(p[0] / 2.0);
    return m2x2(c, -std::polar(1.0, p[2]) * s, std::polar(1.0, p[1]) * s, std::polar(1.0, p[1] + p[2]) * c);
  }
  Mat m(nm == "ccx" ? 3 : 2);
  if (nm == "cx") {  // bit 0 control, bit 1 target
    m.at(0, 0) = 1.0;
    m.at(2, 2) = 1.0;
    m.at(3, 1) = 1.0;
    m.at(1, 3) = 1.0;
  } else if (nm == "cz") {
    m.at(0, 0) = m.at(1, 1) = m.at(2, 2) = 1.0;
    m.at(3, 3) = -1.0;
  } else if (nm == "cp") {
    m.at(0, 0) = m.at(1, 1) = m.at(2, 2) = 1.0;
    m.at(3, 3) = std::polar(1.0, p[0]);
  } else if (nm == "swap") {
    m.at(0, 0) = m.at(3, 3) = 1.0;
    m.at(1, 2) = m.at(2, 1) = 1.0;
  } else if (nm == "ccx") {
    for (size_t in = 0; in < 8; ++in) m.at(((in & 3) == 3) ? (in ^ 4) : in, in) = 1.0;
  } else {
    throw Err(2, "unknown gate name: " + nm);
  }
  return m;
}

static Gate named(const std::string& nm, const std::vector<double>& p, const std::vector<int>& q) {
  const NamedInfo* info = lookup(nm);
  if (!info) throw Err(2, "unknown gate name: " + nm);
  if ((int)q.size() != info->arity) throw Err(2, nm + " expects " + std::to_string(info->arity) + " qubit(s)");
  if ((int)p.size() != info->params) throw Err(2, nm + " expects " + std::to_string(info->params) + " parameter(s)");
  return gate_from_args(named_argorder(nm, p), q, nm, p);
}

// ------------------------------------------------------------- generators ---
// Recipes pinned in DESIGN.md §3 (SPEC.md:170-178 leaves parameters open).
static void add(Circ& c, const std::string& nm, std::vector<double> p, std::vector<int> q) {
  c.g.push_back(named(nm, p, q));
}

static Circ gen(const std::string& kind, int n, int depth, uint64_t seed) {
  if (n < 2 || n > 62) throw Err(2, "benchmark qubit count out of range");
  if (depth < 1 && kind != "qft") throw Err(2, "benchmark depth must be >= 1");
  Circ c;
  c.n = n;
  if (kind == "qft") {
    for (int j = n - 1; j >= 0; --j) {
      add(c, "h", {}, {j});
      for (int m = j - 1; m >= 0; --m) add(c, "cp", {PI / (double)(1ULL << (j - m))}, {m, j});
    }
    for (int i = 0; i < n / 2; ++i) add(c, "swap", {}, {i, n - 1 - i});
  } else if (kind == "rqc") {
    Rng rng(seed);
    int off0 = (int)rng.below(2);
    for (int cy = 0; cy < depth; ++cy) {
      for (int q = 0; q < n; ++q) {
        int r = (int)rng.below(3);
        if (r == 0) add(c, "rx", {PI / 2.0}, {q});
        else if (r == 1) add(c, "ry", {PI / 2.0}, {q});
        else add(c, "t", {}, {q});
      }
      for (int q = (cy + off0) % 2; q + 1 < n; q += 2) add(c, "cz", {}, {q, q + 1});
    }
  } else if (kind == "ala") {
    Rng rng(seed);
    for (int l = 0; l < depth; ++l) {
      for (int q = 0; q < n; ++q) c.g.push_back(gate_from_args(haar_like(1, rng), {q}));
      for (int q = l % 2; q + 1 < n; q += 2) add(c, "cz", {}, {q, q + 1});
    }
  } else if (kind == "qvc") {
    Rng rng(seed);
    for (int l = 0; l < depth; ++l) {
      std::vector<int> perm(n);
      for (int i = 0; i < n; ++i) perm[i] = i;
      for (int i = n - 1; i >= 1; --i) std::swap(perm[i], perm[rng.below((uint64_t)i + 1)]);
      for (int i = 0; i + 1 < n; i += 2) c.g.push_back(gate_from_args(haar_like(2, rng), {perm[i], perm[i + 1]}));
    }
  } else if (kind == "iqp") {
    Rng rng(seed);
    for (int q = 0; q < n; ++q) add(c, "h", {}, {q});
    for (int l = 0; l < depth; ++l) {
      for (int q = 0; q < n; ++q) {
        int r = (int)rng.below(3);
        if (r == 0) add(c, "t", {}, {q});
        else if (r == 1) add(c, "z", {}, {q});
      }
      for (int q = l % 2; q + 1 < n; q += 2)
        if (rng.below(2) == 1) add(c, "cz", {}, {q, q + 1});
    }
    for (int q = 0; q < n; ++q) add(c, "h", {}, {q});
  } else if (kind == "hes") {
    for (int st = 0; st < depth; ++st) {
      for (int i = 0; i + 1 < n; ++i) {
        add(c, "cx", {}, {i, i + 1});
        add(c, "rz", {0.1}, {i + 1});
        add(c, "cx", {}, {i, i + 1});
      }
      for (int q = 0; q < n; ++q) add(c, "rx", {0.1}, {q});
    }
  } else if (kind == "qaoa") {
    if (n % 2 != 0 || n < 4) throw Err(2, "qaoa needs an even qubit count >= 4");
    Rng rng(seed);
    std::vector<std::pair<int, int>> edges;
    for (int attempt = 0;; ++attempt) {
      if (attempt > 100000) throw Err(2, "qaoa graph generation did not converge");
      std::vector<int> stubs;
      for (int v = 0; v < n; ++v)
        for (int j = 0; j < 3; ++j) stubs.push_back(v);
      for (int i = (int)stubs.size() - 1; i >= 1; --i) std::swap(stubs[i], stubs[rng.below((uint64_t)i + 1)]);
      edges.clear();
      std::set<std::pair<int, int>> seen;
      bool ok = true;
      for (size_t i = 0; i + 1 < stubs.size(); i += 2) {
        int a = std::min(stubs[i], stubs[i + 1]), b = std::max(stubs[i], stubs[i + 1]);
        if (a == b || seen.count({a, b})) {
          ok = false;
          break;
        }
        seen.insert({a, b});
        edges.push_back({a, b});
      }
      if (ok) break;
    }
    std::vector<double> gam(depth), bet(depth);
    for (int l = 0; l < depth; ++l) {
      gam[l] = rng.unif(0.0, PI);
      bet[l] = rng.unif(0.0, PI / 2.0);
    }
    for (int q = 0; q < n; ++q) add(c, "h", {}, {q});
    for (int l = 0; l < depth; ++l) {
      for (auto& e : edges) {
        add(c, "cx", {}, {e.first, e.second});
        add(c, "rz", {2.0 * gam[l]}, {e.second});
        add(c, "cx", {}, {e.first, e.second});
      }
      for (int q = 0; q < n; ++q) add(c, "rx", {2.0 * bet[l]}, {q});
    }
  } else {
    throw Err(2, "unknown benchmark kind: " + kind);
  }
  return c;
}

// ------------------------------------------------------------ cost model ---
// SPEC.md:316-323, 357-382, 399.
struct CostRec {
  int k;
  uint64_t ops;
  int threads;
  double spg;
};
struct CostModel {
  std::vector<CostRec> recs;
  int bench_n = 0;
  std::string precision = "f64", host;
};

static CostModel cm_parse(const std::string& text) {
  CostModel cm;
  std::istringstream in(text);
  std::string line;
  int ln = 0;
  bool ver = false;
  while (std::getline(in, line)) {
    ++ln;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.find_first_not_of(" \t") == std::string::npos) continue;
    std::istringstream ls(line);
    std::string head;
    ls >> head;
    if (head == "version") {
      int v = 0;
      ls >> v;
      if (v != 1) throw Err(1, "line " + std::to_string(ln) + ": unsupported cost-model version");
      ver = true;
    } else if (head == "precision") {
      ls >> cm.precision;
    } else if (head == "bench_n") {
      ls >> cm.bench_n;
    } else if (head == "host") {
      std::string rest;
      std::getline(ls, rest);
      size_t st = rest.find_first_not_of(" \t");
      cm.host = st == std::string::npos ? "" : rest.substr(st);
    } else if (head.rfind("k=", 0) == 0) {
      CostRec r{};
      unsigned long long ops = 0;
      if (std::sscanf(line.c_str(), " k=%d ops=%llu threads=%d spg=%lf", &r.k, &ops, &r.threads, &r.spg) != 4)
        throw Err(1, "line " + std::to_string(ln) + ": malformed cost record");
      r.ops = ops;
      if (!(r.spg > 0.0)) throw Err(1, "line " + std::to_string(ln) + ": seconds_per_group must be positive");
      cm.recs.push_back(r);
    } else {
      throw Err(1, "line " + std::to_string(ln) + ": unknown cost-model key '" + head + "'");
    }
  }
  if (!ver) throw Err(1, "cost model missing 'version 1' header");
  return cm;
}

// Linear interpolation of seconds-per-group in log2(op_count) among the
// records of matching (k, threads), clamped at both ends, times 2^(n-k).
static double estimate(const CostModel& cm, int k, uint64_t ops, int threads, int n, bool* ok) {
  std::vector<std::pair<double, double>> pts;
  std::set<uint64_t> have;
  for (auto& r : cm.recs)
    if (r.k == k && r.threads == threads && !have.count(r.ops)) {
      have.insert(r.ops);
      pts.push_back({std::log2((double)std::max<uint64_t>(r.ops, 1)), r.spg});
    }
  if (pts.empty()) {
    *ok = false;
    return 0.0;
  }
  std::stable_sort(pts.begin(), pts.end(), [](auto& a, auto& b) { return a.first < b.first; });
  *ok = true;
  double x = std::log2((double)std::max<uint64_t>(ops, 1));
  double spg;
  if (x <= pts.front().first) spg = pts.front().second;
  else if (x >= pts.back().first) spg = pts.back().second;
  else {
    size_t i = 0;
    while (!(pts[i].first <= x && x <= pts[i + 1].first)) ++i;
    double f = (x - pts[i].first) / (pts[i + 1].first - pts[i].first);
    spg = pts[i].second + (pts[i + 1].second - pts[i].second) * f;
  }
  return spg * std::ldexp(1.0, n - k);
}

// ------------------------------------------------------- tile and fusion ---
// CircuitTile + Algorithm 1 with the
// ambiguities pinned as in DESIGN.md §4.
struct FuseCfg {
  int mode = 1;  // 0 none, 1 size-only, 2 adaptive
  int k_max = 5;
  int64_t max_ops = -1;
  bool agglom = true, multi = true;
  double zt = 1e-8, ot = 1e-8;
  int max_trav = 64;
  int threads = 1;  // thread-count column used for cost lookups
};

struct Blk {
  int id;
  std::vector<int> gates;
  std::vector<int> wires;
  bool mat_ok = false;
  Gate mat;
  int64_t ops = -1;
};

struct Fuser {
  const Circ& C;
  FuseCfg cfg;
  const CostModel* cm;
  int n;
  std::vector<std::vector<int>> rows;  // cell = block id or -1
  std::map<int, Blk> blocks;
  int next_id = 0;

  Fuser(const Circ& c, const FuseCfg& f, const CostModel* m) : C(c), cfg(f), cm(m), n(c.n) {}

  int row_of(int id) const {
    const Blk& b = blocks.at(id);
    for (size_t r = 0; r < rows.size(); ++r)
      if (rows[r][b.wires[0]] == id) return (int)r;
    throw Err(3, "tile corrupted");
  }
  bool free_in(size_t r, const std::vector<int>& w) const {
    for (int q : w)
      if (rows[r][q] != -1) return false;
    return true;
  }
  void put(size_t r, int id) {
    for (int q : blocks[id].wires) rows[r][q] = id;
  }
  void clear(size_t r, int id) {
    for (int q : blocks[id].wires) rows[r][q] = -1;
  }

  void build() {
    std::vector<int> last(n, -1);
    for (size_t i = 0; i < C.g.size(); ++i) {
      Blk b;
      b.id = next_id++;
      b.gates = {(int)i};
      b.wires = C.g[i].t;
      int r = 0;
      for (int q : b.wires) r = std::max(r, last[q] + 1);
      while ((int)rows.size() <= r) rows.push_back(std::vector<int>(n, -1));
      blocks[b.id] = b;
      put(r, b.id);
      for (int q : b.wires) last[q] = r;
    }
  }

  // left fold of the constituent gates, starting from `base` when given
  Gate fold(const std::vector<int>& gates, size_t from, const Gate* base) {
    Gate acc = base ? *base : C.g[gates[0]];
    for (size_t i = base ? from : 1; i < gates.size(); ++i) acc = fuse2(acc, C.g[gates[i]]);
    return acc;
  }
  void materialize(Blk& b) {
    if (b.mat_ok) return;
    b.mat = fold(b.gates, 0, nullptr);
    b.mat_ok = true;
  }
  int64_t ops_of(Blk& b) {
    if (b.ops < 0) {
      materialize(b);
      b.ops = (int64_t)profile_of(b.mat.m, cfg.zt, cfg.ot).ops;
    }
    return b.ops;
  }

  // fusibility of first (earlier) and second; on success for adaptive mode
  // the materialized product is returned through *prod.
  bool fusible(Blk& a, Blk& b, int k, Gate* prod, bool* have) {
    *have = false;
    std::vector<int> u = wires_union(a.wires, b.wires);
    if ((int)u.size() > k) return false;
    if (cfg.mode != 2) return true;
    materialize(a);
    *prod = fold(b.gates, 0, &a.mat);
    *have = true;
    int64_t ops = (int64_t)profile_of(prod->m, cfg.zt, cfg.ot).ops;
    if (cfg.max_ops >= 0 && ops > cfg.max_ops) return false;
    if (!cm) throw Err(2, "adaptive fusion needs a cost model");
    bool o1, o2, o3;
    double cf = estimate(*cm, (int)u.size(), (uint64_t)ops, cfg.threads, n, &o1);
    double ca = estimate(*cm, (int)a.wires.size(), (uint64_t)ops_of(a), cfg.threads, n, &o2);
    double cb = estimate(*cm, (int)b.wires.size(), (uint64_t)ops_of(b), cfg.threads, n, &o3);
    if (!o1 || !o2 || !o3) return false;
    return cf <= ca + cb;
  }

  // remove a (row ra) and b (row rb), create the fused block, place it.
  // r = the upper of the two rows; placement r+1, then r, else new row r+1.
  void fuse(int ida, int idb, size_t r, Gate* prod, bool have) {
    Blk& a = blocks[ida];
    Blk& b = blocks[idb];
    Blk c;
    c.id = next_id++;
    c.gates = a.gates;
    c.gates.insert(c.gates.end(), b.gates.begin(), b.gates.end());
    c.wires = wires_union(a.wires, b.wires);
    if (have) {
      c.mat = std::move(*prod);
      c.mat_ok = true;
    }
    int ra = row_of(ida), rb = row_of(idb);
    clear(ra, ida);
    clear(rb, idb);
    blocks.erase(ida);
    blocks.erase(idb);
    int cid = c.id;
    blocks[cid] = std::move(c);
    const std::vector<int>& w = blocks[cid].wires;
    if (r + 1 < rows.size() && free_in(r + 1, w)) put(r + 1, cid);
    else if (free_in(r, w)) put(r, cid);
    else {
      rows.insert(rows.begin() + (long)r + 1, std::vector<int>(n, -1));
      put(r + 1, cid);
    }
  }

  void compress() {
    bool moved = true;
    while (moved) {
      moved = false;
      for (int r = (int)rows.size() - 2; r >= 0; --r) {
        for (int q = 0; q < n; ++q) {
          int id = rows[r][q];
          if (id < 0 || blocks[id].wires[0] != q) continue;
          if (free_in(r + 1, blocks[id].wires)) {
            clear(r, id);
            put(r + 1, id);
            moved = true;
          }
        }
      }
    }
    std::vector<std::vector<int>> keep;
    for (auto& row : rows) {
      bool any = false;
      for (int v : row) any = any || v >= 0;
      if (any) keep.push_back(row);
    }
    rows.swap(keep);
  }

  bool traverse(int k) {
    bool delta = false;
    std::set<std::pair<int, int>> tried;
    for (size_t r = 0; r < rows.size(); ++r) {
      for (int q = 0; q < n && r < rows.size(); ++q) {
        int top = rows[r][q];
        if (top < 0 || r + 1 >= rows.size()) continue;
        if (free_in(r + 1, blocks[top].wires)) {  // MoveDown into vacancy
          clear(r, top);
          put(r + 1, top);
          continue;
        }
        int bot = rows[r + 1][q];
        if (bot < 0 || tried.count({top, bot})) continue;
        tried.insert({top, bot});
        Gate prod;
        bool have = false;
        if (fusible(blocks[top], blocks[bot], k, &prod, &have)) {
          fuse(top, bot, r, &prod, have);
          delta = true;
        }
      }
      for (int q = 1; q < n && r < rows.size(); ++q) {
        int a = rows[r][q - 1], b = rows[r][q];
        if (a < 0 || b < 0 || a == b) continue;
        std::pair<int, int> key(std::min(a, b), std::max(a, b));
        if (tried.count(key)) continue;
        tried.insert(key);
        int first = blocks[a].wires[0] < blocks[b].wires[0] ? a : b;
        int second = first == a ? b : a;
        Gate prod;
        bool have = false;
        if (fusible(blocks[first], blocks[second], k, &prod, &have)) {
          fuse(first, second, r, &prod, have);
          delta = true;
        }
      }
    }
    compress();
    return delta;
  }

  Circ flatten() {
    Circ out;
    out.n = n;
    for (auto& row : rows) {
      std::vector<int> ids;
      for (int q = 0; q < n; ++q) {
        int id = row[q];
        if (id >= 0 && blocks[id].wires[0] == q) ids.push_back(id);
      }
      for (int id : ids) {
        Blk& b = blocks[id];
        if (b.gates.size() == 1) out.g.push_back(C.g[b.gates[0]]);
        else {
          materialize(b);
          Gate g = b.mat;
          g.name.clear();
          g.p.clear();
          out.g.push_back(g);
        }
      }
    }
    return out;
  }
};

struct FuseStats {
  int64_t orig = 0, fused = 0, total_ops = 0;
  double ratio = 1.0, wall = 0.0;
};

static Circ run_fusion(const Circ& c, const FuseCfg& cfg, const CostModel* cm, FuseStats* st) {
  auto t0 = std::chrono::steady_clock::now();
  if (cfg.k_max < 1 || cfg.k_max > 12) throw Err(2, "k_max must be in [1, 12]");
  if (cfg.mode == 2 && !cm) throw Err(2, "adaptive fusion needs a cost model");
  Circ out;
  if (cfg.mode == 0) out = c;
  else {
    Fuser f(c, cfg, cm);
    f.build();
    int k0 = cfg.agglom ? std::min(2, cfg.k_max) : cfg.k_max;
    for (int k = k0; k <= cfg.k_max; ++k)
      for (int it = 0; it < cfg.max_trav; ++it)
        if (!f.traverse(k) || !cfg.multi) break;
    out = f.flatten();
  }
  st->orig = (int64_t)c.g.size();
  st->fused = (int64_t)out.g.size();
  st->ratio = st->fused > 0 ? (double)st->orig / (double)st->fused : 1.0;
  st->total_ops = 0;
  for (auto& g : out.g) st->total_ops += (int64_t)profile_of(g.m, cfg.zt, cfg.ot).ops;
  st->wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

// ---------------------------------------------------------------- kernel ---
// SPEC.md:407-498.
struct Split {
  int s = 0, kL = 0, kH = 0, ell = 0;
  std::vector<int> lo, hi, red;
};

static Split split_targets(const std::vector<int>& t, int s) {
  Split sp;
  sp.s = s;
  for (int x = 0; (int)sp.red.size() < s; ++x)
    if (!std::binary_search(t.begin(), t.end(), x)) sp.red.push_back(x);
  int maxred = s > 0 ? sp.red.back() : -1;
  for (int q : t) (q < maxred ? sp.lo : sp.hi).push_back(q);
  sp.kL = (int)sp.lo.size();
  sp.kH = (int)sp.hi.size();
  sp.ell = sp.kL + s;
  return sp;
}

static std::vector<uint64_t> masks_for(const Split& sp, int n) {
  int width = n - (int)(sp.lo.size() + sp.hi.size()) - sp.s;
  std::vector<uint64_t> m(sp.kH + 1, 0);
  for (int i = 0; i <= sp.kH; ++i) {
    int lo = (i == 0 ? -1 : sp.hi[i - 1] - sp.ell) - i + 1;
    int hi = (i == sp.kH) ? width : sp.hi[i] - sp.ell - i;
    for (int b = std::max(lo, 0); b < std::min(hi, width); ++b) m[i] |= 1ULL << b;
  }
  return m;
}

struct EntryOp {
  uint32_t row, col;
  uint8_t kre, kim;
  double re, im;
};

struct Plan {
  int n, k, s;
  std::vector<int> t;
  Split sp;
  std::vector<uint64_t> masks;
  std::vector<EntryOp> ops;          // row-major, both-Zero entries excluded
  std::vector<uint32_t> row_begin;   // CSR over ops
  std::vector<uint8_t> kre, kim;     // full kind table (for override checks)
  bool runtime = false;
  Mat m;
};

static Plan make_plan(const Gate& g, int n, int s, double zt, double ot, bool runtime) {
  int k = (int)g.t.size();
  if (s < 0) throw Err(2, "s must be >= 0");
  if (k + s > n) throw Err(2, "gate size plus SIMD exponent exceeds qubit count");
  Plan p;
  p.n = n;
  p.k = k;
  p.s = s;
  p.t = g.t;
  p.sp = split_targets(g.t, s);
  p.masks = masks_for(p.sp, n);
  Profile pr = profile_of(g.m, zt, ot);
  p.kre = pr.kre;
  p.kim = pr.kim;
  p.runtime = runtime;
  p.m = g.m;
  size_t d = g.m.dim();
  for (size_t r = 0; r < d; ++r) {
    p.row_begin.push_back((uint32_t)p.ops.size());
    for (size_t c = 0; c < d; ++c) {
      size_t i = r * d + c;
      if (pr.kre[i] == K_ZERO && pr.kim[i] == K_ZERO) continue;
      p.ops.push_back({(uint32_t)r, (uint32_t)c, pr.kre[i], pr.kim[i], g.m.e[i].real(), g.m.e[i].imag()});
    }
  }
  p.row_begin.push_back((uint32_t)p.ops.size());
  return p;
}

static inline uint64_t start_index(uint64_t t, const std::vector<uint64_t>& masks) {
  uint64_t v = 0;
  for (size_t i = 0; i < masks.size(); ++i) v += (t & masks[i]) << i;
  return v;
}

// one real scalar's contribution, lowered per its kind
template <typename R>
static inline void acc_entry(uint8_t kr, uint8_t ki, R mr, R mi, R xr, R xi, R& yr, R& yi) {
  switch (kr) {
    case K_ONE: yr += xr; yi += xi; break;
    case K_MONE: yr -= xr; yi -= xi; break;
    case K_GEN: yr += mr * xr; yi += mr * xi; break;
    default: break;
  }
  switch (ki) {
    case K_ONE: yr -= xi; yi += xr; break;
    case K_MONE: yr += xi; yi -= xr; break;
    case K_GEN: yr -= mi * xi; yi += mi * xr; break;
    default: break;
  }
}

// apply_kernel over [tb, te) of the 2^(n-k-s) loop counter.  Each counter
// value covers 2^s lanes; lane-inner loops are what SIMD width s buys.
template <typename R>
static void apply_range(const Plan& p, R* re, R* im, const Mat* over, uint64_t tb, uint64_t te) {
  const int k = p.k, s = p.s, ell = p.sp.ell;
  const size_t D = (size_t)1 << k, S = (size_t)1 << s;
  // offsets of the 2^k group elements inside the lower region, per lane
  std::vector<uint64_t> loff(D * S), hoff(D);
  for (size_t j = 0; j < D; ++j) {
    uint64_t lo = 0, hi = 0;
    for (int b = 0; b < p.sp.kL; ++b) lo |= ((j >> b) & 1ULL) << p.sp.lo[b];
    for (int b = 0; b < p.sp.kH; ++b) hi |= ((j >> (p.sp.kL + b)) & 1ULL) << (p.sp.hi[b] - ell);
    hoff[j] = hi;
    for (size_t l = 0; l < S; ++l) {
      uint64_t lane = 0;
      for (int b = 0; b < s; ++b) lane |= ((l >> b) & 1ULL) << p.sp.red[b];
      loff[j * S + l] = lo | lane;
    }
  }
  std::vector<EntryOp> ops = p.ops;
  if (over) {
    for (auto& e : ops) {
      const cd& v = over->at(e.row, e.col);
      e.re = v.real();
      e.im = v.imag();
    }
  }
  std::vector<R> mr(ops.size()), mi(ops.size());
  for (size_t i = 0; i < ops.size(); ++i) {
    mr[i] = (R)ops[i].re;
    mi[i] = (R)ops[i].im;
  }
  std::vector<R> xr(D * S), xi(D * S), yr(D * S), yi(D * S);
  std::vector<uint64_t> idx(D * S);
  for (uint64_t t = tb; t < te; ++t) {
    uint64_t v = start_index(t, p.masks);
    for (size_t j = 0; j < D; ++j) {  // gather
      uint64_t base = (v | hoff[j]) << ell;
      for (size_t l = 0; l < S; ++l) {
        uint64_t a = base | loff[j * S + l];
        idx[j * S + l] = a;
        xr[j * S + l] = re[a];
        xi[j * S + l] = im[a];
      }
    }
    for (size_t r = 0; r < D; ++r) {  // sparse matvec, lanes innermost
      R* orr = &yr[r * S];
      R* oii = &yi[r * S];
      for (size_t l = 0; l < S; ++l) orr[l] = oii[l] = (R)0;
      for (uint32_t e = p.row_begin[r]; e < p.row_begin[r + 1]; ++e) {
        const EntryOp& op = ops[e];
        const R* pr = &xr[op.col * S];
        const R* pi = &xi[op.col * S];
        for (size_t l = 0; l < S; ++l) acc_entry<R>(op.kre, op.kim, mr[e], mi[e], pr[l], pi[l], orr[l], oii[l]);
      }
    }
    for (size_t q = 0; q < D * S; ++q) {  // scatter
      re[idx[q]] = yr[q];
      im[idx[q]] = yi[q];
    }
  }
}

// dense, unspecialised matvec over the ORIGINAL matrix
template <typename R>
static void reference_apply(const Gate& g, int n, R* re, R* im) {
  int k = (int)g.t.size();
  size_t D = (size_t)1 << k;
  uint64_t groups = 1ULL << (n - k);
  std::vector<R> xr(D), xi(D);
  std::vector<uint64_t> off(D);
  for (size_t j = 0; j < D; ++j) off[j] = scatter_bits(j, g.t);
  for (uint64_t t = 0; t < groups; ++t) {
    uint64_t base = t;
    for (int b = 0; b < k; ++b) {
      uint64_t lowm = (1ULL << g.t[b]) - 1;
      base = ((base & ~lowm) << 1) | (base & lowm);
    }
    for (size_t j = 0; j < D; ++j) {
      xr[j] = re[base | off[j]];
      xi[j] = im[base | off[j]];
    }
    for (size_t r = 0; r < D; ++r) {
      R yr = 0, yi = 0;
      for (size_t c = 0; c < D; ++c) {
        R ar = (R)g.m.at(r, c).real(), ai = (R)g.m.at(r, c).imag();
        yr += ar * xr[c] - ai * xi[c];
        yi += ar * xi[c] + ai * xr[c];
      }
      re[base | off[r]] = yr;
      im[base | off[r]] = yi;
    }
  }
}

// ------------------------------------------------------------------- sim ---
// run_circuit: plan each gate, split [0, 2^(n-k-s)) into
// `threads` contiguous chunks (remainder to the last), barrier per gate.
// The group range [lo, hi) of one gate (the whole [0, T) in run_circuit;
// one stratum of it in the bench's bounded CPU sample) split over threads.
template <typename R>
static void apply_threads(const Plan& p, R* re, R* im, const Mat* over, int threads, uint64_t lo, uint64_t hi) {
  if (threads <= 1) {
    apply_range<R>(p, re, im, over, lo, hi);
    return;
  }
  uint64_t chunk = (hi - lo) / (uint64_t)threads;
  std::vector<std::thread> pool;
  for (int i = 0; i < threads; ++i) {
    uint64_t b = lo + chunk * (uint64_t)i;
    uint64_t e = (i + 1 == threads) ? hi : lo + chunk * (uint64_t)(i + 1);
    if (b < e) pool.emplace_back([&, b, e] { apply_range<R>(p, re, im, over, b, e); });
  }
  for (auto& th : pool) th.join();
}

template <typename R>
static void apply_threads(const Plan& p, R* re, R* im, const Mat* over, int threads) {
  apply_threads<R>(p, re, im, over, threads, 0, 1ULL << (p.n - p.k - p.s));
}

// Every gate of the circuit over stratum `slice` of `n_slices` equal parts of
// its group range: the same per-gate work pattern as run_circuit on a 1/n_slices
// sample of every gate (bench.py's bounded CPU baseline; not a simulation).
template <typename R>
static void run_circ_slice(const Circ& c, R* re, R* im, int threads, int s, double zt, double ot, uint64_t slice,
                           uint64_t n_slices, double* t_plan, double* t_exec) {
  double tp = 0, te = 0;
  for (const Gate& g : c.g) {
    auto a = std::chrono::steady_clock::now();
    Plan p = make_plan(g, c.n, s, zt, ot, false);
    auto b = std::chrono::steady_clock::now();
    const uint64_t T = 1ULL << (p.n - p.k - p.s);
    const uint64_t ns = std::min<uint64_t>(n_slices, T), sl = slice % ns;
    apply_threads<R>(p, re, im, nullptr, threads, T / ns * sl, sl + 1 == ns ? T : T / ns * (sl + 1));
    auto e = std::chrono::steady_clock::now();
    tp += std::chrono::duration<double>(b - a).count();
    te += std::chrono::duration<double>(e - b).count();
  }
  *t_plan = tp;
  *t_exec = te;
}

template <typename R>
static double run_circ(const Circ& c, R* re, R* im, int threads, int s, double zt, double ot, double* t_plan,
                       double* t_exec, int g_begin, int g_end) {
  double tp = 0, te = 0;
  if (g_end < 0 || g_end > (int)c.g.size()) g_end = (int)c.g.size();
  for (int i = g_begin; i < g_end; ++i) {
    auto a = std::chrono::steady_clock::now();
    Plan p = make_plan(c.g[i], c.n, s, zt, ot, false);
    auto b = std::chrono::steady_clock::now();
    apply_threads<R>(p, re, im, nullptr, threads);
    auto e = std::chrono::steady_clock::now();
    tp += std::chrono::duration<double>(b - a).count();
    te += std::chrono::duration<double>(e - b).count();
  }
  if (t_plan) *t_plan = tp;
  if (t_exec) *t_exec = te;
  return tp + te;
}

template <typename R>
static double norm_kahan(const R* re, const R* im, uint64_t N) {
  double sum = 0.0, comp = 0.0;
  for (uint64_t i = 0; i < N; ++i) {
    double x = (double)re[i], y = (double)im[i];
    double term = x * x + y * y - comp;
    double t = sum + term;
    comp = (t - sum) - term;
    sum = t;
  }
  return std::sqrt(sum);
}

}  // namespace orc

// =============================================================== C API ====
using namespace orc;

static thread_local std::string g_err;
static int fail(const std::exception& e) {
  g_err = e.what();
  if (auto* x = dynamic_cast<const Err*>(&e)) return x->code;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 2;
  return 3;
}
#define GUARD(...)                                \
  try {                                           \
    __VA_ARGS__;                                  \
    return 0;                                     \
  } catch (const std::exception& e) { return fail(e); }

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---- circuits
void* orc_circuit_new(int n) {
  Circ* c = new Circ();
  c->n = n;
  return c;
}
void orc_circuit_free(void* c) { delete (Circ*)c; }
int orc_circuit_add_named(void* c, const char* name, const double* p, int np, const int* q, int nq) {
  GUARD({
    Circ* C = (Circ*)c;
    for (int i = 0; i < nq; ++i)
      if (q[i] < 0 || q[i] >= C->n) throw Err(1, "qubit index out of range");
    C->g.push_back(named(name, std::vector<double>(p, p + np), std::vector<int>(q, q + nq)));
  })
}
// m: 2*4^k doubles, interleaved re/im, row-major, argument order
int orc_circuit_add_matrix(void* c, int k, const int* q, const double* m) {
  GUARD({
    Circ* C = (Circ*)c;
    Mat M(k);
    for (size_t i = 0; i < M.e.size(); ++i) M.e[i] = cd(m[2 * i], m[2 * i + 1]);
    C->g.push_back(gate_from_args(M, std::vector<int>(q, q + k)));
  })
}
int orc_circuit_n_qubits(void* c) { return ((Circ*)c)->n; }
int orc_circuit_n_gates(void* c) { return (int)((Circ*)c)->g.size(); }
int orc_circuit_gate_k(void* c, int i) { return (int)((Circ*)c)->g[i].t.size(); }
void orc_circuit_gate_targets(void* c, int i, int* out) {
  auto& g = ((Circ*)c)->g[i];
  for (size_t j = 0; j < g.t.size(); ++j) out[j] = g.t[j];
}
void orc_circuit_gate_matrix(void* c, int i, double* out) {
  auto& g = ((Circ*)c)->g[i];
  for (size_t j = 0; j < g.m.e.size(); ++j) {
    out[2 * j] = g.m.e[j].real();
    out[2 * j + 1] = g.m.e[j].imag();
  }
}
const char* orc_circuit_gate_name(void* c, int i) { return ((Circ*)c)->g[i].name.c_str(); }

int orc_gen_benchmark(const char* kind, int n, int depth, uint64_t seed, void** out) {
  GUARD({ *out = new Circ(gen(kind, n, depth, seed)); })
}

// ---- gatecore primitives (matrices as interleaved re/im)
int orc_random_unitary(int k, uint64_t seed, int skip, double* out) {
  GUARD({
    Rng rng(seed);
    for (int i = 0; i < skip; ++i) haar_like(k, rng);
    Mat m = haar_like(k, rng);
    for (size_t j = 0; j < m.e.size(); ++j) {
      out[2 * j] = m.e[j].real();
      out[2 * j + 1] = m.e[j].imag();
    }
  })
}
void orc_prng_stream(uint64_t seed, int count, uint64_t* u, double* normals) {
  Rng a(seed), b(seed);
  for (int i = 0; i < count; ++i) u[i] = a.u64();
  for (int i = 0; i < count; ++i) normals[i] = b.gauss();
}
int orc_classify(double x, double zt, double ot) { return kind_of(x, zt, ot); }
// kinds_out: 2*4^k (re kind, im kind per entry); counts: gen, one, mone, ops
int orc_profile(int k, const double* m, double zt, double ot, uint8_t* kinds_out, uint64_t* counts) {
  GUARD({
    Mat M(k);
    for (size_t i = 0; i < M.e.size(); ++i) M.e[i] = cd(m[2 * i], m[2 * i + 1]);
    Profile p = profile_of(M, zt, ot);
    if (kinds_out)
      for (size_t i = 0; i < M.e.size(); ++i) {
        kinds_out[2 * i] = p.kre[i];
        kinds_out[2 * i + 1] = p.kim[i];
      }
    counts[0] = p.gen;
    counts[1] = p.one;
    counts[2] = p.mone;
    counts[3] = p.ops;
  })
}
int orc_is_unitary(int k, const double* m, double tol) {
  Mat M(k);
  for (size_t i = 0; i < M.e.size(); ++i) M.e[i] = cd(m[2 * i], m[2 * i + 1]);
  return unitary(M, tol) ? 1 : 0;
}
// fuse two sorted-target gates; out_t gets the union, out_m its matrix
int orc_fuse(int k1, const int* t1, const double* m1, int k2, const int* t2, const double* m2, int* out_k, int* out_t,
             double* out_m) {
  GUARD({
    Gate a, b;
    a.m = Mat(k1);
    b.m = Mat(k2);
    a.t.assign(t1, t1 + k1);
    b.t.assign(t2, t2 + k2);
    for (size_t i = 0; i < a.m.e.size(); ++i) a.m.e[i] = cd(m1[2 * i], m1[2 * i + 1]);
    for (size_t i = 0; i < b.m.e.size(); ++i) b.m.e[i] = cd(m2[2 * i], m2[2 * i + 1]);
    Gate f = fuse2(a, b);
    *out_k = (int)f.t.size();
    for (size_t i = 0; i < f.t.size(); ++i) out_t[i] = f.t[i];
    for (size_t i = 0; i < f.m.e.size(); ++i) {
      out_m[2 * i] = f.m.e[i].real();
      out_m[2 * i + 1] = f.m.e[i].imag();
    }
  })
}
int orc_expand(int k, const int* t, const double* m, int ku, const int* tu, double* out_m) {
  GUARD({
    Gate g;
    g.m = Mat(k);
    g.t.assign(t, t + k);
    for (size_t i = 0; i < g.m.e.size(); ++i) g.m.e[i] = cd(m[2 * i], m[2 * i + 1]);
    Mat e = embed(g, std::vector<int>(tu, tu + ku));
    for (size_t i = 0; i < e.e.size(); ++i) {
      out_m[2 * i] = e.e[i].real();
      out_m[2 * i + 1] = e.e[i].imag();
    }
  })
}

// ---- kernel plan pieces
// out: [kL, kH, ell, lo..., hi...]
int orc_split(int k, const int* t, int s, int* out) {
  GUARD({
    Split sp = split_targets(std::vector<int>(t, t + k), s);
    out[0] = sp.kL;
    out[1] = sp.kH;
    out[2] = sp.ell;
    int j = 3;
    for (int q : sp.lo) out[j++] = q;
    for (int q : sp.hi) out[j++] = q;
  })
}
int orc_masks(int k, const int* t, int s, int n, uint64_t* out, int* n_out) {
  GUARD({
    Split sp = split_targets(std::vector<int>(t, t + k), s);
    auto m = masks_for(sp, n);
    *n_out = (int)m.size();
    for (size_t i = 0; i < m.size(); ++i) out[i] = m[i];
  })
}
// every amplitude index touched, in loop order: out has 2^n entries
int orc_enumerate_indices(int k, const int* t, int s, int n, uint64_t* out) {
  GUARD({
    Split sp = split_targets(std::vector<int>(t, t + k), s);
    if (k + s > n) throw Err(2, "gate size plus SIMD exponent exceeds qubit count");
    auto masks = masks_for(sp, n);
    uint64_t T = 1ULL << (n - k - s), w = 0;
    size_t D = (size_t)1 << k, S = (size_t)1 << s;
    for (uint64_t tt = 0; tt < T; ++tt) {
      uint64_t v = start_index(tt, masks);
      for (size_t j = 0; j < D; ++j) {
        uint64_t lo = 0, hi = 0;
        for (int b = 0; b < sp.kL; ++b) lo |= ((j >> b) & 1ULL) << sp.lo[b];
        for (int b = 0; b < sp.kH; ++b) hi |= ((j >> (sp.kL + b)) & 1ULL) << (sp.hi[b] - sp.ell);
        for (size_t l = 0; l < S; ++l) {
          uint64_t lane = 0;
          for (int b = 0; b < s; ++b) lane |= ((l >> b) & 1ULL) << sp.red[b];
          out[w++] = ((v | hi) << sp.ell) | lo | lane;
        }
      }
    }
  })
}
// entry count of a plan (entries whose two scalars are not both Zero)
int orc_plan_entry_count(int k, const double* m, double zt, double ot, int* out) {
  GUARD({
    Gate g;
    g.m = Mat(k);
    for (size_t i = 0; i < g.m.e.size(); ++i) g.m.e[i] = cd(m[2 * i], m[2 * i + 1]);
    for (int i = 0; i < k; ++i) g.t.push_back(i);
    Plan p = make_plan(g, k, 0, zt, ot, false);
    *out = (int)p.ops.size();
  })
}

// ---- state application.  prec 64: re/im are double*, prec 32: float*.
// override: NULL or a 2*4^k matrix whose kinds must match the plan's.
int orc_apply(int n, int k, const int* t, const double* m, int s, double zt, double ot, const double* over, void* re,
              void* im, int prec, uint64_t tb, uint64_t te) {
  GUARD({
    Gate g;
    g.m = Mat(k);
    g.t.assign(t, t + k);
    for (size_t i = 0; i < g.m.e.size(); ++i) g.m.e[i] = cd(m[2 * i], m[2 * i + 1]);
    Plan p = make_plan(g, n, s, zt, ot, over != nullptr);
    uint64_t T = 1ULL << (n - k - s);
    if (tb > te || te > T) throw Err(3, "loop range outside [0, 2^(n-k-s))");
    Mat O;
    if (over) {
      O = Mat(k);
      for (size_t i = 0; i < O.e.size(); ++i) {
        O.e[i] = cd(over[2 * i], over[2 * i + 1]);
        if (kind_of(O.e[i].real(), zt, ot) != p.kre[i] || kind_of(O.e[i].imag(), zt, ot) != p.kim[i])
          throw Err(3, "override matrix does not match the planned sparsity pattern");
      }
    }
    if (prec == 64) apply_range<double>(p, (double*)re, (double*)im, over ? &O : nullptr, tb, te);
    else apply_range<float>(p, (float*)re, (float*)im, over ? &O : nullptr, tb, te);
  })
}
int orc_reference_apply(int n, int k, const int* t, const double* m, void* re, void* im, int prec) {
  GUARD({
    Gate g;
    g.m = Mat(k);
    g.t.assign(t, t + k);
    for (size_t i = 0; i < g.m.e.size(); ++i) g.m.e[i] = cd(m[2 * i], m[2 * i + 1]);
    if (prec == 64) reference_apply<double>(g, n, (double*)re, (double*)im);
    else reference_apply<float>(g, n, (float*)re, (float*)im);
  })
}
// runs gates [g_begin, g_end) (g_end < 0: all); times[0]=plan s, times[1]=exec s
int orc_run_circuit(void* c, void* re, void* im, int prec, int threads, int s, double zt, double ot, int g_begin,
                    int g_end, double* times) {
  GUARD({
    Circ* C = (Circ*)c;
    double tp = 0, te = 0;
    if (prec == 64) run_circ<double>(*C, (double*)re, (double*)im, threads, s, zt, ot, &tp, &te, g_begin, g_end);
    else run_circ<float>(*C, (float*)re, (float*)im, threads, s, zt, ot, &tp, &te, g_begin, g_end);
    if (times) {
      times[0] = tp;
      times[1] = te;
    }
  })
}
// every gate over stratum `slice` of `n_slices` of its group range
// (bench.py's bounded CPU sample); times[0]=plan s, times[1]=exec s
int orc_run_circuit_slice(void* c, void* re, void* im, int prec, int threads, int s, double zt, double ot,
                          uint64_t slice, uint64_t n_slices, double* times) {
  GUARD({
    Circ* C = (Circ*)c;
    if (n_slices == 0) throw Err(2, "n_slices must be positive");
    if (prec == 64) run_circ_slice<double>(*C, (double*)re, (double*)im, threads, s, zt, ot, slice, n_slices, &times[0], &times[1]);
    else run_circ_slice<float>(*C, (float*)re, (float*)im, threads, s, zt, ot, slice, n_slices, &times[0], &times[1]);
  })
}
// unfused dense oracle run over a circuit
int orc_reference_run(void* c, void* re, void* im, int prec) {
  GUARD({
    Circ* C = (Circ*)c;
    for (auto& g : C->g) {
      if (prec == 64) reference_apply<double>(g, C->n, (double*)re, (double*)im);
      else reference_apply<float>(g, C->n, (float*)re, (float*)im);
    }
  })
}
double orc_norm(const void* re, const void* im, uint64_t N, int prec) {
  if (prec == 64) return norm_kahan<double>((const double*)re, (const double*)im, N);
  return norm_kahan<float>((const float*)re, (const float*)im, N);
}
double orc_compare(const double* ar, const double* ai, const double* br, const double* bi, uint64_t N) {
  double mx = 0.0;
  for (uint64_t i = 0; i < N; ++i) {
    double dr = ar[i] - br[i], di = ai[i] - bi[i];
    mx = std::max(mx, std::sqrt(dr * dr + di * di));
  }
  return mx;
}

// ---- fusion.  cfg_i: [mode, k_max, agglom, multi, max_trav, threads]
// cfg_d: [zt, ot]; max_ops < 0: unset.  stats: [orig, fused, total_ops]
// stats_d: [ratio, wall_seconds]
int orc_run_fusion(void* c, const int* cfg_i, int64_t max_ops, const double* cfg_d, void* cm, void** out,
                   int64_t* stats, double* stats_d) {
  GUARD({
    FuseCfg f;
    f.mode = cfg_i[0];
    f.k_max = cfg_i[1];
    f.agglom = cfg_i[2] != 0;
    f.multi = cfg_i[3] != 0;
    f.max_trav = cfg_i[4];
    f.threads = cfg_i[5];
    f.max_ops = max_ops;
    f.zt = cfg_d[0];
    f.ot = cfg_d[1];
    FuseStats st;
    Circ r = run_fusion(*(Circ*)c, f, (const CostModel*)cm, &st);
    *out = new Circ(std::move(r));
    stats[0] = st.orig;
    stats[1] = st.fused;
    stats[2] = st.total_ops;
    stats_d[0] = st.ratio;
    stats_d[1] = st.wall;
  })
}
int orc_cost_model_parse(const char* text, void** out) {
  GUARD({ *out = new CostModel(cm_parse(text)); })
}
void orc_cost_model_free(void* cm) { delete (CostModel*)cm; }
int orc_estimate_cost(void* cm, int k, uint64_t ops, int threads, int n, double* out) {
  GUARD({
    bool ok = false;
    *out = estimate(*(CostModel*)cm, k, ops, threads, n, &ok);
    if (!ok) throw Err(2, "no cost records for this gate size / thread count");
  })
}

}  // extern "C"
