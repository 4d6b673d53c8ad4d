// Kernel plans: qubit split, startIdx masks, sparsity-classified entry list
// and the B200 launch structure derived from them.
#include <algorithm>
#include <sstream>

#include "tilesim/plan.hpp"

namespace tilesim {

const char* to_string(KernelClass k) {
  switch (k) {
    case KernelClass::Identity: return "identity";
    case KernelClass::Diagonal: return "diagonal";
    case KernelClass::Direct: return "direct";
    case KernelClass::Tile: return "tile";
  }
  return "?";
}

// Fig. 6 colouring: targets blue, the s smallest other indices red; the lower
// side is everything up to the largest red index (empty when s = 0).
QubitSplit split_qubits(const std::vector<int>& targets, int s) {
  QubitSplit sp;
  sp.s = s;
  for (int x = 0; static_cast<int>(sp.red.size()) < s; ++x)
    if (!std::binary_search(targets.begin(), targets.end(), x)) sp.red.push_back(x);
  const int top_red = s > 0 ? sp.red.back() : -1;
  for (int q : targets) (q < top_red ? sp.lower : sp.higher).push_back(q);
  sp.k_L = static_cast<int>(sp.lower.size());
  sp.k_H = static_cast<int>(sp.higher.size());
  sp.lower_region_size = sp.k_L + s;
  return sp;
}

// masks[i] = bits [p_{i-1} - i + 1, p_i - i) of t, with p the higher targets
// re-indexed into vector space (minus k_L + s), p_{-1} = -1, p_{k_H} = +inf.
MaskTable build_masks(const QubitSplit& sp, int n) {
  const int width = n - sp.k_L - sp.k_H - sp.s;
  const int shift = sp.lower_region_size;
  MaskTable mt;
  mt.masks.assign(sp.k_H + 1, 0);
  int from = 0;
  for (int i = 0; i <= sp.k_H; ++i) {
    const int to = i < sp.k_H ? sp.higher[i] - shift - i : width;
    for (int b = from; b < to && b < width; ++b) mt.masks[i] |= uint64_t{1} << b;
    from = std::max(from, to);
  }
  return mt;
}

uint64_t start_index(uint64_t t, const MaskTable& m) {
  uint64_t v = 0;
  for (size_t i = 0; i < m.masks.size(); ++i) v += (t & m.masks[i]) << i;
  return v;
}

namespace {

bool is_exact(double x, double v) { return x == v; }

// snapped scalar pair of entry i of `m` under the plan's kinds
cplx snapped(const GateMatrix& m, const SparsityProfile& prof, size_t i) {
  return cplx(snap_scalar(m.entries()[i].real(), prof.kinds[i].re), snap_scalar(m.entries()[i].imag(), prof.kinds[i].im));
}

}  // namespace

LaunchStructure derive_launch(const KernelPlan& plan, const GateMatrix* over, int precision_bits) {
  const GateMatrix& src = over ? *over : plan.gate.matrix;
  const int k = plan.gate.k();
  const uint64_t D = uint64_t{1} << k;
  if (over) {
    if (over->k() != k) throw SimError("override matrix size does not match the plan");
    for (size_t i = 0; i < src.entries().size(); ++i) {
      if (classify_scalar(src.entries()[i].real(), plan.zero_tol, plan.one_tol) != plan.profile.kinds[i].re ||
          classify_scalar(src.entries()[i].imag(), plan.zero_tol, plan.one_tol) != plan.profile.kinds[i].im)
        throw SimError("override matrix does not match the planned sparsity pattern");
    }
  }
  std::vector<cplx> S(D * D);
  for (size_t i = 0; i < S.size(); ++i) S[i] = snapped(src, plan.profile, i);
  auto ident = [&](uint64_t r, uint64_t c) {
    return is_exact(S[r * D + c].real(), r == c ? 1.0 : 0.0) && is_exact(S[r * D + c].imag(), 0.0);
  };

  // A local bit b is a control with active value v when every entry whose row
  // or column has bit b == !v is the identity entry.  Peeling all controls
  // leaves the sub-block on rows/cols with every control at its active value.
  LaunchStructure ls;
  uint64_t ctrl_mask = 0, ctrl_val = 0;
  for (int b = 0; b < k; ++b) {
    for (int v = 1; v >= 0; --v) {
      bool ok = true;
      for (uint64_t r = 0; r < D && ok; ++r)
        for (uint64_t c = 0; c < D && ok; ++c) {
          const bool inactive = (((r >> b) & 1u) != static_cast<unsigned>(v)) || (((c >> b) & 1u) != static_cast<unsigned>(v));
          if (inactive && !ident(r, c)) ok = false;
        }
      if (ok) {
        ctrl_mask |= uint64_t{1} << b;
        ctrl_val |= static_cast<uint64_t>(v) << b;
        break;
      }
    }
  }
  std::vector<int> sub_bits;
  for (int b = 0; b < k; ++b) {
    if ((ctrl_mask >> b) & 1u) {
      ls.controls.push_back(plan.gate.targets[b]);
      ls.control_values |= ((ctrl_val >> b) & 1u) << plan.gate.targets[b];
    } else {
      sub_bits.push_back(b);
      ls.sub_targets.push_back(plan.gate.targets[b]);
    }
  }
  ls.ks = static_cast<int>(sub_bits.size());
  const uint64_t d = uint64_t{1} << ls.ks;
  ls.offsets.resize(d);
  std::vector<uint64_t> local(d);  // sub index -> local (gate) index with controls active
  for (uint64_t j = 0; j < d; ++j) {
    uint64_t loc = ctrl_val, q = 0;
    for (int b = 0; b < ls.ks; ++b) {
      loc |= ((j >> b) & 1u) << sub_bits[b];
      q |= ((j >> b) & 1u) << ls.sub_targets[b];
    }
    local[j] = loc;
    ls.offsets[j] = q;
  }
  ls.sub_re.resize(d * d);
  ls.sub_im.resize(d * d);
  bool diagonal = true, identity = true;
  for (uint64_t r = 0; r < d; ++r)
    for (uint64_t c = 0; c < d; ++c) {
      const cplx v = S[local[r] * D + local[c]];
      ls.sub_re[r * d + c] = v.real();
      ls.sub_im[r * d + c] = v.imag();
      ls.nonzero_scalars += (v.real() != 0.0) + (v.imag() != 0.0);
      if (r != c && (v.real() != 0.0 || v.imag() != 0.0)) diagonal = false;
      if (!(v.real() == (r == c ? 1.0 : 0.0) && v.imag() == 0.0)) identity = false;
    }
  const int direct_max = precision_bits == 64 ? 4 : 5;
  if (identity) ls.klass = KernelClass::Identity;
  else if (diagonal) ls.klass = KernelClass::Diagonal;
  else if (ls.ks <= direct_max) ls.klass = KernelClass::Direct;
  else ls.klass = KernelClass::Tile;
  if (ls.ks > 6 && ls.klass != KernelClass::Identity && ls.klass != KernelClass::Diagonal)
    throw ConfigError("GPU kernels support non-diagonal sub-gates of at most 6 qubits (got " + std::to_string(ls.ks) + ")");
  // zero-skipping pays once at least a quarter of the dense scalars are zero
  ls.sparse = ls.nonzero_scalars * 4 <= 3 * (2 * d * d);
  return ls;
}

KernelPlan plan_kernel(const Gate& g, int n, int s, double zero_tol, double one_tol, bool runtime_matrix) {
  const int k = g.k();
  if (s < 0) throw ConfigError("SIMD exponent s must be >= 0");
  if (k < 1) throw ConfigError("gate has no targets");
  if (g.targets.back() >= n) throw ConfigError("gate target outside the statevector");
  if (k + s > n) throw ConfigError("gate size plus SIMD exponent exceeds the qubit count");
  KernelPlan p;
  p.gate = g;
  p.n = n;
  p.zero_tol = zero_tol;
  p.one_tol = one_tol;
  p.runtime_matrix = runtime_matrix;
  p.split = split_qubits(g.targets, s);
  p.mask_table = build_masks(p.split, n);
  p.group_masks = s == 0 ? p.mask_table : build_masks(split_qubits(g.targets, 0), n);
  p.profile = sparsity_profile(g.matrix, zero_tol, one_tol);
  const uint64_t D = g.matrix.dim();
  for (uint64_t r = 0; r < D; ++r)
    for (uint64_t c = 0; c < D; ++c) {
      const auto& kp = p.profile.kinds[r * D + c];
      if (kp.re == ScalarKind::Zero && kp.im == ScalarKind::Zero) continue;
      const cplx& v = g.matrix.at(r, c);
      p.entry_ops.push_back({static_cast<uint32_t>(r), static_cast<uint32_t>(c), kp.re, kp.im, v.real(), v.imag()});
    }
  p.launch = derive_launch(p, nullptr, 64);
  return p;
}

std::string describe(const KernelPlan& p) {
  std::ostringstream os;
  os << "targets";
  for (int q : p.gate.targets) os << ' ' << q;
  os << "\nsplit s=" << p.split.s << " k_L=" << p.split.k_L << " k_H=" << p.split.k_H << "\nmasks";
  for (uint64_t m : p.mask_table.masks) {
    os << " 0b";
    bool lead = true;
    for (int b = 63; b >= 0; --b) {
      const bool bit = (m >> b) & 1u;
      if (bit) lead = false;
      if (!lead) os << (bit ? '1' : '0');
    }
    if (lead) os << '0';
  }
  os << "\nentries " << p.entry_ops.size() << " op_count " << p.profile.op_count << "\nkernel "
     << to_string(p.launch.klass) << " ks=" << p.launch.ks << " controls=" << p.launch.controls.size() << "\n";
  for (const EntryOp& e : p.entry_ops)
    os << e.row << ',' << e.col << ' ' << to_string(e.re_kind) << '/' << to_string(e.im_kind) << "\n";
  return os.str();
}

}  // namespace tilesim
