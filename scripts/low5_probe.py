"""[0..4] dense 5-qubit complex128 launches: RQC-30 fused gate 8 vs a random
dense unitary, on a random and on a basis state (design measurement)."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2503_19894_b200 as ts
from tests._util import random_gate_matrix
os.environ["TSG_NO_PASS"] = "1"
f, _ = ts.run_fusion(ts.gen_benchmark("rqc", 30, 20, 42), ts.FusionConfig(k_max=5))
g8 = f.gate(8)
mats = {"rqc8": np.asarray(g8.matrix), "rand": random_gate_matrix(5, 5, "dense")}
m = mats["rqc8"]
print("rqc8 targets", list(g8.targets), "abs min", np.abs(m).min(), "zeros", int((m == 0).sum()),
      "re zeros", int((m.real == 0).sum()), "im zeros", int((m.imag == 0).sum()))
for sname in ("random", "basis"):
    sv = ts.Statevector(30, "f64")
    sv.init_random(1) if sname == "random" else sv.init_basis(3)
    for mname, mm in mats.items():
        c = ts.Circuit(30)
        for _ in range(3):
            c.add_matrix([0, 1, 2, 3, 4], mm)
        p = ts.Program(c, "f64")
        p.run(sv, use_graph=False)
        secs, _ = p.run_profiled(sv)
        print(sname, mname, [s["kernel"] for s in p.steps()][0], [round(x * 1e3, 3) for x in secs])
