"""Fidelity of a fused benchmark circuit against the unfused FP64 oracle
(tests/test_gpu_parity.py::test_fused_circuit_matches_oracle, printed)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402
from oracle import binding as ob  # noqa: E402
from tests._util import to_oracle  # noqa: E402

kind, n, depth, prec, kmax = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
c = ts.gen_benchmark(kind, n, depth, 42)
fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
sv = ts.Statevector(n, prec).init_random(1)
re0, im0 = sv.download()
prog = ts.Program(fused, prec)
prog.run(sv)
dt = np.float32 if prec == "f32" else np.float64
ore, oim = re0.astype(dt), im0.astype(dt)
ob.run_circuit(to_oracle(fused), ore, oim, threads=4)
d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
rre, rim = re0.copy(), im0.copy()
ob.reference_run(to_oracle(c), rre, rim)
psi = sv.amplitudes()
fid = abs(np.vdot(rre + 1j * rim, psi)) ** 2
print(f"{os.environ.get('TSG_UMMA', '')}/{os.environ.get('TSG_UMMA_KS', '')} d={d:.3e} 1-fid={1 - fid:.3e} norm={np.linalg.norm(psi):.9f}",
      sorted(set(s['kernel'] for s in prog.steps())))
