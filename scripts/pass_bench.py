"""Micro-cases for the tile-pass kernel (design measurements, not product):
each case is a small synthetic gate list at n=28 whose gates all fit one pass;
prints device ms per pass and the same gates without passes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("PB_ROOT"):  # a variant build of the package (design experiments)
    sys.path.insert(0, os.environ["PB_ROOT"])
import paper_2503_19894_b200 as ts  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

N = int(os.environ.get("PB_N", 28))
PREC = os.environ.get("PB_PREC", "f64")


def case(name, gates):
    if gates in ("rqc", "rqc4"):  # the 5- (4-) qubit fused gates of RQC-n (k <= 5)
        fused, _ = ts.run_fusion(ts.gen_benchmark("rqc", N, 20, 42), ts.FusionConfig(k_max=5))
        c = ts.Circuit(N)
        for g in fused.gates():
            if g.k == (5 if gates == "rqc" else 4):
                c.add_matrix(g.targets, g.matrix)
    else:
        c = ts.Circuit(N)
        for q, kind in gates:
            if kind == "blockdiag2":  # 4-qubit gate mixing its two low qubits, blocks chosen by the two high ones
                rng = np.random.default_rng(sum(q))
                m = np.zeros((16, 16), complex)
                for b in range(4):
                    u = random_gate_matrix(2, int(rng.integers(1000)), "dense")
                    idx = [b * 4 + j for j in range(4)]
                    m[np.ix_(idx, idx)] = u
                c.add_matrix(sorted(q), m)
            else:
                c.add_matrix(sorted(q), random_gate_matrix(len(q), sum(q) * 7 + len(name), kind))
    out = []
    for no_pass in (False, True):
        if no_pass:
            os.environ["TSG_NO_PASS"] = "1"
        elif os.environ.get("PB_FORCE") == "1":  # every eligible gate joins the pass (cost calibration)
            os.environ["TSG_PASS_FORCE"] = "1"
        prog = ts.Program(c, PREC)
        os.environ.pop("TSG_NO_PASS", None)
        os.environ.pop("TSG_PASS_FORCE", None)
        sv = ts.Statevector(N, PREC).init_basis(3)
        prog.run(sv)
        best = min(prog.run(sv)["execution_s"] for _ in range(3))
        out.append((best * 1e3, [s["kernel"] for s in prog.steps()]))
    sweep_ms = 2 * (1 << N) * (16 if PREC == "f64" else 8) / 6.5e12 * 1e3
    print(f"{name:28s} pass {out[0][0]:7.3f} ms  no-pass {out[1][0]:7.3f} ms  (1 sweep at 6.5 TB/s: {sweep_ms:.3f} ms) "
          f"steps {out[0][1]}")


sel = sys.argv[1:] or None
cases = {
    "empty-ish (1 diag T)": [([2, 3], "diag"), ([1, 4], "diag")],
    "2x gen ks1 low": [([1], "dense"), ([3], "dense")],
    "2x gen ks1 high": [([7], "dense"), ([9], "dense")],
    "2x gen ks2": [([6, 7], "dense"), ([8, 9], "dense")],
    "2x gen ks3": [([5, 6, 7], "dense"), ([8, 9, 10], "dense")],
    "2x gen ks4": [([5, 6, 7, 8], "dense"), ([7, 8, 9, 10], "dense")],
    "2x gen ks4 low": [([0, 1, 2, 3], "dense"), ([1, 2, 3, 4], "dense")],
    "8x diag X": [([0, 1, 9, 10], "diag")] * 8,
    "8x diag T": [([0, 1, 20, 21], "diag")] * 8,
    "8x diag I": [([9, 10, 20, 21], "diag")] * 8,
    "8x diag C": [([22, 23, 24, 25], "diag")] * 8,
    "ks5 dense 0-4": [([0, 1, 2, 3, 4], "dense")],
    "ks5 dense 3-7": [([3, 4, 5, 6, 7], "dense")],
    "ks5 dense 5-9": [([5, 6, 7, 8, 9], "dense")],
    "ks5 dense 7-11": [([7, 8, 9, 10, 11], "dense")],
    "ks5 dense 20-24": [([20, 21, 22, 23, 24], "dense")],
    "ks5 diag-ish 7-11": [([7, 8, 9, 10, 11], "controlled")],
    "ks5 rqc-like": "rqc",
    "ks4 rqc-like": "rqc4",
    "4x gen ks2 blk out": [([6, 7, 20, 21], "blockdiag2"), ([8, 9, 22, 23], "blockdiag2"), ([6, 7, 24, 25], "blockdiag2"), ([8, 9, 26, 27], "blockdiag2")],
    "4x gen ks2 blk thr": [([0, 1, 6, 7], "blockdiag2"), ([2, 3, 6, 7], "blockdiag2"), ([0, 1, 8, 9], "blockdiag2"), ([2, 3, 8, 9], "blockdiag2")],
    "4x gen ks2 blk iter": [([6, 7, 9, 10], "blockdiag2"), ([0, 1, 9, 10], "blockdiag2"), ([2, 3, 9, 10], "blockdiag2"), ([7, 8, 9, 10], "blockdiag2")],
    "4x gen ks2 noblk": [([6, 7], "dense"), ([8, 9], "dense"), ([6, 7], "dense"), ([8, 9], "dense")],
    "4x gen ks3 same": [([6, 7, 8], "dense")] * 4,
    "4x gen ks3 diff": [([6, 7, 8], "dense"), ([9, 10, 11], "dense"), ([6, 7, 8], "dense"), ([9, 10, 11], "dense")],
    "4x gen ks1 same-layout": [([6], "dense"), ([7], "dense"), ([8], "dense"), ([6], "dense")],
    "2x gen ks4 smem": [([5, 6, 7, 8], "dense"), ([7, 8, 9, 10], "dense")],
    "1x gen ks4 smem": [([5, 6, 7, 8], "dense")],
    "1x gen ks4 smem low": [([0, 1, 2, 3], "dense")],
    "1x gen ks5 smem": [([5, 6, 7, 8, 9], "dense")],
    "1x gen ks3": [([6, 7, 8], "dense")],
    "1x gen ks3 low": [([1, 2, 3], "dense")],
    "2x ks5 dense": [([5, 6, 7, 8, 9], "dense"), ([7, 8, 9, 10, 11], "dense")],
    "ks5+ks4 dense": [([5, 6, 7, 8, 9], "dense"), ([7, 8, 9, 10], "dense")],
    "3x gen ks4 smem": [([5, 6, 7, 8], "dense"), ([7, 8, 9, 10], "dense"), ([5, 6, 9, 10], "dense")],
    "4x gen ks4 smem": [([5, 6, 7, 8], "dense"), ([7, 8, 9, 10], "dense"), ([5, 6, 9, 10], "dense"), ([6, 7, 8, 9], "dense")],
    "4x perm ks2": [([6, 7], "perm"), ([8, 9], "perm"), ([1, 7], "perm"), ([2, 9], "perm")],
    "4x perm ks4": [([0, 1, 9, 10], "perm"), ([2, 3, 7, 8], "perm"), ([0, 2, 9, 7], "perm"), ([5, 6, 7, 8], "perm")],
}
for k, v in cases.items():
    if sel is None or any(s in k for s in sel):
        case(k, v)
