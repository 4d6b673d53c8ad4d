"""Device time of 5-qubit complex128 gates on a dense random 30-qubit state:
a random dense unitary vs the RQC-30 fused gates on the same targets, each
timed twice in interleaved order (TSG_DMMA_MODE=direct|stream).  Design
measurements."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2503_19894_b200 as ts  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

n = 30
sv = ts.Statevector(n, "f64").init_random(3)
f, _ = ts.run_fusion(ts.gen_benchmark("rqc", n, 20, 42), ts.FusionConfig(k_max=5))
cases = [("dense", [0, 1, 2, 3, 4], random_gate_matrix(5, 5, "dense")),
         ("dense", [7, 8, 9, 10, 11], random_gate_matrix(5, 5, "dense"))]
for g in f.gates():
    if g.targets in ([0, 1, 2, 3, 4], [7, 8, 9, 10, 11]):
        nz = np.count_nonzero(np.abs(g.matrix) > 1e-12) / g.matrix.size
        cases.append((f"rqc nz={nz:.2f}", g.targets, g.matrix))
plans = [(name, tg, ts.KernelPlan(ts.Gate(tg, m), n)) for name, tg, m in cases]
for rep in range(2):
    for name, tg, p in plans:
        ts.apply_kernel(p, sv)
        sv.synchronize()
        sv.timer_begin()
        for _ in range(5):
            ts.apply_kernel(p, sv)
        print(f"rep{rep} {os.environ.get('TSG_DMMA_MODE', 'default'):8s} {name:12s} {tg}: {sv.timer_end() / 5 * 1e3:.3f} ms")
