"""Time a pass built from a slice of a fused benchmark circuit, and the same
slice restricted to its diagonal / non-diagonal gates (which ops cost what).
usage: pass_probe.py KIND N KMAX FIRST COUNT [PREC]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("PB_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_19894_b200 as ts  # noqa: E402

kind, n, kmax, first, count = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
prec = sys.argv[6] if len(sys.argv) > 6 else "f64"
fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, 1 if kind == "qft" else 20, 42), ts.FusionConfig(k_max=kmax))
gates = [fused.gate(i) for i in range(first, first + count)]
sv = ts.Statevector(n, prec).init_basis(3)


def is_diag(g):
    m = np.asarray(g.matrix)
    return np.count_nonzero(m - np.diag(np.diag(m))) == 0


def time_of(sel, label):
    c = ts.Circuit(n)
    for g in sel:
        c.add_matrix(list(g.targets), np.asarray(g.matrix))
    os.environ["TSG_PASS_FORCE"] = "1"
    prog = ts.Program(c, prec)
    os.environ.pop("TSG_PASS_FORCE")
    prog.run(sv)
    best = min(prog.run_profiled(sv)[1]["execution_s"] for _ in range(3))
    print(f"{label:28s} gates {len(sel):3d} steps {[s['kernel'] for s in prog.steps()]} {best * 1e3:8.3f} ms")


for g in gates:
    ls = ts.plan_kernel(g, n).info()
    print("  ", list(g.targets), "diag" if is_diag(g) else "gen", "sub", ls.get("sub_targets"), "ctrl", ls.get("controls"))
time_of(gates, "all")
time_of([g for g in gates if is_diag(g)], "diagonal only")
time_of([g for g in gates if not is_diag(g)], "non-diagonal only")
time_of(gates[:1], "first gate")
