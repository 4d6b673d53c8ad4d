"""Full-state parity at 30 qubits for the families the round-2 paths touch
(beyond tests/test_gpu_fullsize.py): ALA-30 c128 k<=5 (dense class; JIT DMMA
products), HES-30 c64 k<=5 (INT8 tensor-core products, passes), QAOA-30 c64
k<=3 (the commutation-aware planner's plan).  The oracle runs on every host
thread.  usage: fullsize_extra.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402
from oracle import binding as ob  # noqa: E402
from tests._util import to_oracle  # noqa: E402
from tests.test_gpu_fullsize import _host_stats  # noqa: E402

THREADS = os.cpu_count() or 1
n = 30
for kind, depth, seed, k, prec, bar in (("ala", 20, 42, 5, "f64", 1e-10), ("hes", 6, 42, 5, "f32", 1e-5),
                                        ("qaoa", 4, 7, 3, "f32", 1e-5)):
    fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, seed), ts.FusionConfig(k_max=k))
    sv = ts.Statevector(n, prec).init_random(1)
    ore, oim = sv.download()
    dt = np.float64 if prec == "f64" else np.float32
    ore, oim = ore.astype(dt), oim.astype(dt)
    prog = ts.Program(fused, prec)
    prog.run(sv)
    t0 = time.time()
    ob.run_circuit(to_oracle(fused), ore, oim, threads=THREADS)
    t_cpu = time.time() - t0
    mx, l2, fid = _host_stats(sv, ore, oim)
    ok = mx <= bar and fid >= 1 - 1e-9
    print(f"{kind.upper()}-30 {prec} k<={k}: {len(prog.steps())} steps, jit {prog.jit_kernels()}, "
          f"max|dpsi| {mx:.3e}  ||dpsi|| {l2:.3e}  1-F {1 - fid:.3e}  oracle {t_cpu:.0f}s  {'OK' if ok else 'FAIL'}",
          flush=True)
    del prog, sv
