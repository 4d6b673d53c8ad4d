"""GPU debug: k_stream (full-range launches) vs the group-space kernels
(forced by splitting the range in two) over tile geometries, plus timing."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2503_19894_b200 as ts  # noqa: E402
from oracle import binding as ob  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

n = 14
cases = [
    ([0, 1, 2], "dense"), ([0, 1, 2, 3], "controlled"), ([4, 9, 12], "dense"), ([0, 1, 2, 3], "dense"),
    ([1, 2, 3, 13], "controlled"), ([0, 5, 6, 13], "controlled"), ([3, 8, 9, 10], "controlled"),
    ([0, 2, 6, 11], "controlled"), ([8, 9, 10, 11], "controlled"), ([1, 2, 3, 4], "controlled"),
    ([0, 1, 2, 3, 4], "dense"), ([7, 8, 9, 10, 11], "dense"), ([0, 1, 2, 3, 4, 5], "controlled"),
    ([2, 4, 6, 8, 10, 12], "controlled"),
]
for prec in (64, 32):
    for targets, kind in cases:
        k = len(targets)
        m = random_gate_matrix(k, 3, kind)
        rng = np.random.default_rng(0)
        re = rng.standard_normal(1 << n)
        im = rng.standard_normal(1 << n)
        a = ts.Statevector(n, "f64" if prec == 64 else "f32").upload(re, im)
        b = ts.Statevector(n, "f64" if prec == 64 else "f32").upload(re, im)
        p = ts.KernelPlan(ts.Gate(targets, m), n)
        ts.apply_kernel(p, a)
        T = 1 << (n - k)
        ts.apply_kernel(p, b, None, 0, T // 2)
        ts.apply_kernel(p, b, None, T // 2, T)
        d = ts.compare_states(a, b)
        print(prec, targets, kind, p.info()["kernel"], p.info()["sub_k"], f"diff={d:.2e}", flush=True)

for prec in (64, 32):
    N = 28
    for targets in ([20, 21, 22], [20, 21, 22, 23], [20, 21, 22, 23, 24], [0, 1, 2, 3, 4], [0, 6, 12, 18, 24]):
        k = len(targets)
        m = random_gate_matrix(k, 5, "dense")
        sv = ts.Statevector(N, "f64" if prec == 64 else "f32").init_zero()
        p = ts.KernelPlan(ts.Gate(targets, m), N)
        ts.apply_kernel(p, sv)
        sv.synchronize()
        reps = 3
        sv.timer_begin()
        for _ in range(reps):
            ts.apply_kernel(p, sv)
        t = sv.timer_end() / reps
        gb = 2 * (1 << N) * (16 if prec == 64 else 8) / t / 1e9
        print(f"timing prec={prec} n={N} targets={targets} {t*1e3:.3f} ms {gb:.0f} GB/s", flush=True)
