"""Find the first fused gate whose GPU application disagrees with the oracle
(tests/test_gpu_parity.py::test_small_states_every_kernel_path).  usage: debug_small.py N PREC"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402
from oracle import binding as ob  # noqa: E402
from tests._util import random_gate_matrix, to_oracle  # noqa: E402

n, prec = int(sys.argv[1]), int(sys.argv[2])
P = {64: "f64", 32: "f32"}[prec]
rng = np.random.default_rng(n * 10 + prec)
c = ts.Circuit(n)
for i in range(40):
    k = int(rng.integers(1, min(5, n) + 1))
    t = sorted(int(q) for q in rng.choice(n, size=k, replace=False))
    kind = ["dense", "perm", "diag", "controlled"][i % 4] if k > 1 else "dense"
    c.add_matrix(t, random_gate_matrix(k, 700 + i, kind))
fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=5))
sv = ts.Statevector(n, P).init_random(2)
re, im = sv.download()
dt = np.float64 if prec == 64 else np.float32
for gi in range(len(fused)):
    g = fused.gate(gi)
    one = ts.Circuit(n)
    one.add_matrix(list(g.targets), np.asarray(g.matrix))
    prog = ts.Program(one, P)
    s2 = ts.Statevector(n, P).upload(re, im)
    prog.run(s2)
    ore, oim = re.astype(dt), im.astype(dt)
    ob.run_circuit(to_oracle(one), ore, oim)
    d = ts.compare_states(s2, (ore.astype(np.float64), oim.astype(np.float64)))
    info = ts.plan_kernel(g, n).info()
    print(gi, list(g.targets), [s["kernel"] for s in prog.steps()], "sub", info.get("sub_targets"), "ctrl",
          info.get("controls"), f"d={d:.2e}")
    re, im = s2.download()
