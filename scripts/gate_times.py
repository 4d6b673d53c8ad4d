"""Per-gate device time of a fused circuit with each gate's targets, sub-gate
size, DMMA element order and nonzero fraction.  usage: gate_times.py KIND N DEPTH PREC KMAX"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402

kind, n, depth, prec, kmax = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 42), ts.FusionConfig(k_max=kmax))
prog = ts.Program(fused, prec)
sv = ts.Statevector(n, prec).init_zero()
prog.run(sv)
secs, _ = prog.run_profiled(sv)
for st in prog.steps():
    g = fused.gate(st["first_gate"])
    m = np.asarray(g.matrix)
    info = ts.plan_kernel(g, n).info()
    nz = np.count_nonzero(np.abs(m) > 1e-12) / m.size
    print(f"{st['kernel']:30s} t={list(g.targets)} ctrl={info.get('controls')} sub={info.get('sub_targets')} "
          f"nz={nz:.2f} {secs[st['first_gate']] * 1e3:7.3f} ms")
