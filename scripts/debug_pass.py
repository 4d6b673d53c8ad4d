"""Debug helper: find the first gate prefix where the tile-pass program
disagrees with the same program without passes.  usage: debug_pass.py KIND N DEPTH PREC KMAX"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402

kind, n, depth, prec, kmax = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 42), ts.FusionConfig(k_max=kmax))
gates = fused.gates()
rng = np.random.default_rng(3)
re0, im0 = rng.standard_normal(1 << n), rng.standard_normal(1 << n)
nrm = np.sqrt((re0 ** 2 + im0 ** 2).sum())
re0, im0 = re0 / nrm, im0 / nrm


def run(count, no_pass):
    c = ts.Circuit(n)
    for g in gates[:count]:
        c.add_matrix(g.targets, g.matrix)
    if no_pass:
        os.environ["TSG_NO_PASS"] = "1"
    prog = ts.Program(c, prec)
    os.environ.pop("TSG_NO_PASS", None)
    sv = ts.Statevector(n, prec).upload(re0, im0)
    prog.run(sv)
    return sv, prog


lo, hi = 0, len(gates)
sv, _ = run(hi, False)
ref, _ = run(hi, True)
print("full diff", ts.compare_states(sv, ref))
while hi - lo > 1:
    mid = (lo + hi) // 2
    a, _ = run(mid, False)
    b, _ = run(mid, True)
    d = ts.compare_states(a, b)
    if d > 1e-4:
        hi = mid
    else:
        lo = mid
print("first bad prefix", hi)
os.environ["TSG_PASS_DEBUG"] = "1"
a, prog = run(hi, False)
for st in prog.steps():
    print(st)
for g in gates[max(0, hi - 3):hi]:
    m = np.asarray(g.matrix)
    r, c = np.nonzero(np.abs(m) > 1e-8)
    print("gate", g.targets, "mixed", bin(np.bitwise_or.reduce(r ^ c)), ts.plan_kernel(g, n).info())
