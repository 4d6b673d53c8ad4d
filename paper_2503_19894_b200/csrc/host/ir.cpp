// Circuit IR: named-gate table (proj/src/circuit.cpp:25-148 semantics), the
// line-oriented text format (reference parser circuit.cpp:225-455)
// and the benchmark generators (recipes pinned in DESIGN.md).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <set>
#include <sstream>

#include "tilesim/ir.hpp"

namespace tilesim {

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kHalfSqrt2 = 0.70710678118654752440084436210485;

struct NamedSpec {
  const char* name;
  int arity;
  int nparams;
};
constexpr NamedSpec kTable[] = {
    {"x", 1, 0},   {"y", 1, 0},  {"z", 1, 0},  {"h", 1, 0},    {"s", 1, 0},   {"sdg", 1, 0},
    {"t", 1, 0},   {"tdg", 1, 0}, {"rx", 1, 1}, {"ry", 1, 1},   {"rz", 1, 1},  {"u3", 1, 3},
    {"cx", 2, 0},  {"cz", 2, 0},  {"cp", 2, 1}, {"swap", 2, 0}, {"ccx", 3, 0},
};

const NamedSpec* spec_of(const std::string& name) {
  for (const NamedSpec& s : kTable)
    if (name == s.name) return &s;
  return nullptr;
}

GateMatrix one_qubit(cplx m00, cplx m01, cplx m10, cplx m11) {
  GateMatrix m(1);
  m.entries() = {m00, m01, m10, m11};
  return m;
}

// matrix with index bit j = j-th argument qubit
GateMatrix argument_order_matrix(const std::string& name, const std::vector<double>& p) {
  const cplx i1(0.0, 1.0);
  if (name == "h") return one_qubit(kHalfSqrt2, kHalfSqrt2, kHalfSqrt2, -kHalfSqrt2);
  if (name == "x") return one_qubit(0.0, 1.0, 1.0, 0.0);
  if (name == "y") return one_qubit(0.0, -i1, i1, 0.0);
  if (name == "z") return one_qubit(1.0, 0.0, 0.0, -1.0);
  if (name == "s") return one_qubit(1.0, 0.0, 0.0, i1);
  if (name == "sdg") return one_qubit(1.0, 0.0, 0.0, -i1);
  if (name == "t") return one_qubit(1.0, 0.0, 0.0, std::polar(1.0, kPi / 4.0));
  if (name == "tdg") return one_qubit(1.0, 0.0, 0.0, std::polar(1.0, -kPi / 4.0));
  if (name == "rx" || name == "ry" || name == "u3") {
    const double c = std::cos(p[0] / 2.0), s = std::sin(p[0] / 2.0);
    if (name == "rx") return one_qubit(c, -i1 * s, -i1 * s, c);
    if (name == "ry") return one_qubit(c, -s, s, c);
    return one_qubit(c, -std::polar(1.0, p[2]) * s, std::polar(1.0, p[1]) * s, std::polar(1.0, p[1] + p[2]) * c);
  }
  if (name == "rz") return one_qubit(std::polar(1.0, -p[0] / 2.0), 0.0, 0.0, std::polar(1.0, p[0] / 2.0));
  if (name == "ccx") {  // bits 0,1 control, bit 2 target
    GateMatrix m(3);
    for (uint64_t col = 0; col < 8; ++col) m.at((col & 3) == 3 ? col ^ 4 : col, col) = 1.0;
    return m;
  }
  GateMatrix m(2);
  if (name == "cx") {  // bit 0 control, bit 1 target
    m.at(0, 0) = m.at(2, 2) = 1.0;
    m.at(1, 3) = m.at(3, 1) = 1.0;
  } else if (name == "swap") {
    m.at(0, 0) = m.at(3, 3) = 1.0;
    m.at(1, 2) = m.at(2, 1) = 1.0;
  } else if (name == "cz" || name == "cp") {
    m.at(0, 0) = m.at(1, 1) = m.at(2, 2) = 1.0;
    m.at(3, 3) = name == "cz" ? cplx(-1.0, 0.0) : std::polar(1.0, p[0]);
  } else {
    throw std::invalid_argument("unknown gate name: " + name);
  }
  return m;
}

}  // namespace

int named_gate_arity(const std::string& name) {
  const NamedSpec* s = spec_of(name);
  return s ? s->arity : 0;
}

int named_gate_param_count(const std::string& name) {
  const NamedSpec* s = spec_of(name);
  return s ? s->nparams : 0;
}

Gate make_named_gate(const std::string& name, const std::vector<double>& params, const std::vector<int>& qubits) {
  const NamedSpec* s = spec_of(name);
  if (!s) throw std::invalid_argument("unknown gate name: " + name);
  if (static_cast<int>(qubits.size()) != s->arity)
    throw std::invalid_argument(name + " expects " + std::to_string(s->arity) + " qubit(s)");
  if (static_cast<int>(params.size()) != s->nparams)
    throw std::invalid_argument(name + " expects " + std::to_string(s->nparams) + " parameter(s)");
  return make_gate_arg_order(argument_order_matrix(name, params), qubits, name, params);
}

// ------------------------------------------------------------------ parser
namespace {

std::string drop_comment(const std::string& raw) {
  std::string s = raw.substr(0, raw.find('#'));
  if (!s.empty() && s.back() == '\r') s.pop_back();
  return s;
}

bool is_blank(const std::string& s) { return s.find_first_not_of(" \t") == std::string::npos; }

// whitespace tokenizer with 1-based columns
class Tokens {
 public:
  Tokens(const std::string& s, int line) : s_(s), line_(line) {}
  std::string next(int* col) {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t')) ++i_;
    *col = static_cast<int>(i_) + 1;
    const size_t b = i_;
    while (i_ < s_.size() && s_[i_] != ' ' && s_[i_] != '\t') ++i_;
    return s_.substr(b, i_ - b);
  }
  bool done() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t')) ++i_;
    return i_ >= s_.size();
  }
  int column() const { return static_cast<int>(i_) + 1; }
  int line() const { return line_; }

 private:
  const std::string& s_;
  int line_;
  size_t i_ = 0;
};

long to_long(const std::string& tok, int line, int col, const char* what) {
  char* end = nullptr;
  const long v = std::strtol(tok.c_str(), &end, 10);
  if (tok.empty() || end != tok.c_str() + tok.size())
    throw ParseError(std::string("expected ") + what + ", got '" + tok + "'", line, col);
  return v;
}

double to_double(const std::string& tok, int line, int col) {
  char* end = nullptr;
  const double v = std::strtod(tok.c_str(), &end);
  if (tok.empty() || end != tok.c_str() + tok.size()) throw ParseError("expected a number, got '" + tok + "'", line, col);
  return v;
}

int to_qubit(const std::string& tok, int n, int line, int col) {
  const long q = to_long(tok, line, col, "a qubit index");
  if (q < 0 || q >= n)
    throw ParseError("qubit index " + std::to_string(q) + " out of range for " + std::to_string(n) + " qubit(s)", line,
                     col);
  return static_cast<int>(q);
}

std::string g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

}  // namespace

Circuit parse_circuit(const std::string& text) {
  std::vector<std::string> lines;
  {
    std::string cur;
    for (char ch : text) {
      if (ch == '\n') {
        lines.push_back(cur);
        cur.clear();
      } else {
        cur += ch;
      }
    }
    if (!cur.empty()) lines.push_back(cur);
  }
  size_t li = 0;
  // index of the next non-blank line (after comment removal), or -1
  auto next_line = [&](bool required, const char* expect) -> long {
    for (; li < lines.size(); ++li)
      if (!is_blank(drop_comment(lines[li]))) return static_cast<long>(li);
    if (required)
      throw ParseError(std::string("unexpected end of input, expected ") + expect, static_cast<int>(lines.size()) + 1);
    return -1;
  };

  Circuit c;
  const long hdr = next_line(true, "'qubits <n>' header");
  {
    ++li;
    const std::string body = drop_comment(lines[hdr]);
    Tokens tk(body, static_cast<int>(hdr) + 1);
    int col = 0;
    if (tk.next(&col) != "qubits") throw ParseError("file must start with 'qubits <n>'", tk.line(), col);
    const std::string ntok = tk.next(&col);
    const long n = to_long(ntok, tk.line(), col, "a qubit count");
    if (n < 1 || n > 62) throw ParseError("qubit count must be in [1, 62]", tk.line(), col);
    if (!tk.done()) throw ParseError("trailing tokens after qubit count", tk.line(), tk.column());
    c.n_qubits = static_cast<int>(n);
  }

  for (long at = next_line(false, ""); at >= 0; at = next_line(false, "")) {
    ++li;
    const std::string body = drop_comment(lines[at]);
    const int ln = static_cast<int>(at) + 1;
    Tokens tk(body, ln);
    int col = 0;
    const std::string head = tk.next(&col);
    if (head == "qubits") throw ParseError("duplicate 'qubits' header", ln, col);

    if (head == "matrix") {
      int kcol = 0;
      const std::string ktok = tk.next(&kcol);
      const long k = to_long(ktok, ln, kcol, "a gate size");
      if (k < 1 || k > kFusedQubitCap)
        throw ParseError("matrix gate size must be in [1, " + std::to_string(kFusedQubitCap) + "]", ln, kcol);
      std::vector<int> qs;
      for (long j = 0; j < k; ++j) {
        int qcol = 0;
        const std::string qt = tk.next(&qcol);
        qs.push_back(to_qubit(qt, c.n_qubits, ln, qcol));
      }
      if (!tk.done()) throw ParseError("trailing tokens after matrix header", ln, tk.column());
      GateMatrix m(static_cast<int>(k));
      for (uint64_t r = 0; r < m.dim(); ++r) {
        const long rl = next_line(true, "a matrix row");
        ++li;
        const std::string row = drop_comment(lines[rl]);
        Tokens rt(row, static_cast<int>(rl) + 1);
        for (uint64_t cc = 0; cc < m.dim(); ++cc) {
          int ecol = 0;
          const std::string tok = rt.next(&ecol);
          const size_t comma = tok.find(',');
          if (comma == std::string::npos) throw ParseError("expected 're,im' entry", rt.line(), ecol);
          const double re = to_double(tok.substr(0, comma), rt.line(), ecol);
          const double im = to_double(tok.substr(comma + 1), rt.line(), ecol + static_cast<int>(comma) + 1);
          m.at(r, cc) = cplx(re, im);
        }
        if (!rt.done()) throw ParseError("too many entries in matrix row", rt.line(), rt.column());
      }
      if (!m.finite()) throw ParseError("matrix has non-finite entries", ln, col);
      if (!is_unitary(m, 1e-10)) throw ParseError("matrix is not unitary (tolerance 1e-10)", ln, col);
      try {
        c.gates.push_back(make_gate_arg_order(m, qs));
      } catch (const std::invalid_argument& e) {
        throw ParseError(e.what(), ln, col);
      }
      continue;
    }

    std::string name = head;
    std::vector<double> params;
    const size_t lp = head.find('(');
    if (lp != std::string::npos) {
      if (head.back() != ')') throw ParseError("unterminated parameter list", ln, col + static_cast<int>(head.size()));
      name = head.substr(0, lp);
      const std::string list = head.substr(lp + 1, head.size() - lp - 2);
      const int base = col + static_cast<int>(lp) + 1;
      size_t from = 0;
      for (;;) {
        const size_t comma = list.find(',', from);
        params.push_back(to_double(list.substr(from, comma == std::string::npos ? std::string::npos : comma - from), ln,
                                   base + static_cast<int>(from)));
        if (comma == std::string::npos) break;
        from = comma + 1;
      }
    }
    const NamedSpec* s = spec_of(name);
    if (!s) throw ParseError("unknown gate name '" + name + "'", ln, col);
    if (static_cast<int>(params.size()) != s->nparams)
      throw ParseError(name + " expects " + std::to_string(s->nparams) + " parameter(s), got " +
                           std::to_string(params.size()),
                       ln, col);
    std::vector<int> qs;
    for (int j = 0; j < s->arity; ++j) {
      int qcol = 0;
      const std::string qt = tk.next(&qcol);
      if (qt.empty()) throw ParseError(name + " expects " + std::to_string(s->arity) + " qubit(s)", ln, qcol);
      qs.push_back(to_qubit(qt, c.n_qubits, ln, qcol));
    }
    if (!tk.done()) throw ParseError("trailing tokens after gate line", ln, tk.column());
    try {
      c.gates.push_back(make_named_gate(name, params, qs));
    } catch (const std::invalid_argument& e) {
      throw ParseError(e.what(), ln, col);
    }
  }
  return c;
}

// Named gates are emitted with their sorted targets (as the reference does,
// circuit.cpp:416-419).  For cx/ccx whose argument order is not sorted this
// does not round-trip; we keep the reference's output.
std::string serialize_circuit(const Circuit& c) {
  std::ostringstream os;
  os << "qubits " << c.n_qubits << "\n";
  for (const Gate& g : c.gates) {
    if (g.name.empty()) {
      os << "matrix " << g.k();
      for (int q : g.targets) os << ' ' << q;
      os << '\n';
      for (uint64_t r = 0; r < g.matrix.dim(); ++r) {
        for (uint64_t cc = 0; cc < g.matrix.dim(); ++cc)
          os << (cc ? " " : "") << g17(g.matrix.at(r, cc).real()) << ',' << g17(g.matrix.at(r, cc).imag());
        os << '\n';
      }
      continue;
    }
    os << g.name;
    for (size_t j = 0; j < g.params.size(); ++j) os << (j ? ',' : '(') << g17(g.params[j]);
    if (!g.params.empty()) os << ')';
    for (int q : g.targets) os << ' ' << q;
    os << '\n';
  }
  return os.str();
}

Circuit load_circuit_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open circuit file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return parse_circuit(ss.str());
}

void save_circuit_file(const Circuit& c, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw SimError("cannot write circuit file: " + path);
  out << serialize_circuit(c);
}

// --------------------------------------------------------------- generators
BenchmarkKind parse_benchmark_kind(const std::string& s) {
  static const std::pair<const char*, BenchmarkKind> kinds[] = {
      {"qft", BenchmarkKind::QFT}, {"ala", BenchmarkKind::ALA}, {"rqc", BenchmarkKind::RQC},
      {"qvc", BenchmarkKind::QVC}, {"iqp", BenchmarkKind::IQP}, {"hes", BenchmarkKind::HES},
      {"qaoa", BenchmarkKind::QAOA}};
  for (const auto& k : kinds)
    if (s == k.first) return k.second;
  throw ConfigError("unknown benchmark kind: " + s);
}

namespace {
struct Builder {
  Circuit c;
  void named(const char* nm, std::vector<int> q, std::vector<double> p = {}) {
    c.gates.push_back(make_named_gate(nm, p, q));
  }
  void raw(const GateMatrix& m, std::vector<int> q) { c.gates.push_back(make_gate_arg_order(m, q)); }
};

// random 3-regular graph: configuration model, reject self-loops and
// multi-edges, edges kept in pairing order as (min, max)
std::vector<std::pair<int, int>> cubic_graph(int n, Prng& rng) {
  for (int attempt = 0; attempt <= 100000; ++attempt) {
    std::vector<int> stub;
    stub.reserve(3 * n);
    for (int v = 0; v < n; ++v) stub.insert(stub.end(), 3, v);
    for (int i = static_cast<int>(stub.size()) - 1; i > 0; --i) std::swap(stub[i], stub[rng.next_below(i + 1)]);
    std::vector<std::pair<int, int>> e;
    std::set<std::pair<int, int>> seen;
    bool simple = true;
    for (size_t i = 0; simple && i + 1 < stub.size(); i += 2) {
      const std::pair<int, int> ed(std::min(stub[i], stub[i + 1]), std::max(stub[i], stub[i + 1]));
      simple = ed.first != ed.second && seen.insert(ed).second;
      e.push_back(ed);
    }
    if (simple) return e;
  }
  throw ConfigError("qaoa graph generation did not converge");
}
}  // namespace

Circuit gen_benchmark(BenchmarkKind kind, int n, int depth, uint64_t seed) {
  if (n < 2 || n > 62) throw ConfigError("benchmark qubit count out of range");
  if (kind != BenchmarkKind::QFT && depth < 1) throw ConfigError("benchmark depth must be >= 1");
  Builder b;
  b.c.n_qubits = n;
  Prng rng(seed);
  switch (kind) {
    case BenchmarkKind::QFT:  // H then controlled phases to lower qubits, top-down; final swaps
      for (int hi = n - 1; hi >= 0; --hi) {
        b.named("h", {hi});
        for (int lo = hi - 1; lo >= 0; --lo) b.named("cp", {lo, hi}, {kPi / static_cast<double>(uint64_t{1} << (hi - lo))});
      }
      for (int i = 0; i < n / 2; ++i) b.named("swap", {i, n - 1 - i});
      break;
    case BenchmarkKind::RQC: {
      const int parity = static_cast<int>(rng.next_below(2));
      for (int cyc = 0; cyc < depth; ++cyc) {
        for (int q = 0; q < n; ++q) {
          switch (rng.next_below(3)) {
            case 0: b.named("rx", {q}, {kPi / 2.0}); break;
            case 1: b.named("ry", {q}, {kPi / 2.0}); break;
            default: b.named("t", {q}); break;
          }
        }
        for (int q = (cyc + parity) % 2; q + 1 < n; q += 2) b.named("cz", {q, q + 1});
      }
      break;
    }
    case BenchmarkKind::ALA:
      for (int layer = 0; layer < depth; ++layer) {
        for (int q = 0; q < n; ++q) b.raw(random_unitary(1, rng), {q});
        for (int q = layer % 2; q + 1 < n; q += 2) b.named("cz", {q, q + 1});
      }
      break;
    case BenchmarkKind::QVC:
      for (int layer = 0; layer < depth; ++layer) {
        std::vector<int> perm(n);
        for (int i = 0; i < n; ++i) perm[i] = i;
        for (int i = n - 1; i > 0; --i) std::swap(perm[i], perm[rng.next_below(i + 1)]);
        for (int i = 0; i + 1 < n; i += 2) b.raw(random_unitary(2, rng), {perm[i], perm[i + 1]});
      }
      break;
    case BenchmarkKind::IQP:
      for (int q = 0; q < n; ++q) b.named("h", {q});
      for (int layer = 0; layer < depth; ++layer) {
        for (int q = 0; q < n; ++q) {
          const uint64_t pick = rng.next_below(3);
          if (pick == 0) b.named("t", {q});
          if (pick == 1) b.named("z", {q});
        }
        for (int q = layer % 2; q + 1 < n; q += 2)
          if (rng.next_below(2) == 1) b.named("cz", {q, q + 1});
      }
      for (int q = 0; q < n; ++q) b.named("h", {q});
      break;
    case BenchmarkKind::HES:  // first-order TFIM Trotter steps, J = h = 1, dt = 0.05
      for (int step = 0; step < depth; ++step) {
        for (int i = 0; i + 1 < n; ++i) {
          b.named("cx", {i, i + 1});
          b.named("rz", {i + 1}, {0.1});
          b.named("cx", {i, i + 1});
        }
        for (int q = 0; q < n; ++q) b.named("rx", {q}, {0.1});
      }
      break;
    case BenchmarkKind::QAOA: {  // MaxCut on a random 3-regular graph, p = depth
      if (n % 2 != 0 || n < 4) throw ConfigError("qaoa needs an even qubit count >= 4");
      const auto edges = cubic_graph(n, rng);
      std::vector<double> gamma(depth), beta(depth);
      for (int l = 0; l < depth; ++l) {
        gamma[l] = rng.uniform(0.0, kPi);
        beta[l] = rng.uniform(0.0, kPi / 2.0);
      }
      for (int q = 0; q < n; ++q) b.named("h", {q});
      for (int l = 0; l < depth; ++l) {
        for (const auto& e : edges) {
          b.named("cx", {e.first, e.second});
          b.named("rz", {e.second}, {2.0 * gamma[l]});
          b.named("cx", {e.first, e.second});
        }
        for (int q = 0; q < n; ++q) b.named("rx", {q}, {2.0 * beta[l]});
      }
      break;
    }
  }
  return b.c;
}

}  // namespace tilesim
