"""Every 5-qubit complex128 gate of RQC-30 (k <= 5) timed with the sparse and
the dense DMMA kernel variant (TSG_DMMA_SPARSE) on a dense random state, with
its count of nonzero 8x4 DMMA tiles.  Design measurements."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) == 1:
    for v in ("0", "1"):
        subprocess.run([sys.executable, __file__, v], env=dict(os.environ, TSG_DMMA_SPARSE=v), check=True)
    sys.exit(0)
import numpy as np  # noqa: E402

import paper_2503_19894_b200 as ts  # noqa: E402

n = 30
sv = ts.Statevector(n, "f64").init_random(3)
f, _ = ts.run_fusion(ts.gen_benchmark("rqc", n, 20, 42), ts.FusionConfig(k_max=5))
for i, g in enumerate(f.gates()):
    p = ts.KernelPlan(g, n)
    info = p.info()
    if info["sub_k"] != 5:
        continue
    m = np.asarray(g.matrix)
    re0 = np.count_nonzero(np.abs(m.real) > 1e-8) / m.size
    im0 = np.count_nonzero(np.abs(m.imag) > 1e-8) / m.size
    ts.apply_kernel(p, sv)
    sv.synchronize()
    sv.timer_begin()
    for _ in range(3):
        ts.apply_kernel(p, sv)
    print(f"sparse={sys.argv[1]} gate {i:3d} {g.targets} re-nz {re0:.2f} im-nz {im0:.2f}: {sv.timer_end() / 3 * 1e3:.3f} ms")
