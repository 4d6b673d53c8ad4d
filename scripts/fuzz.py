"""Long randomised parity run (tests/test_gpu_fuzz.py's generator, many seeds,
optional forced passes).  usage: fuzz.py FIRST_SEED COUNT [NMAX]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402
from oracle import binding as ob  # noqa: E402
from tests._util import to_oracle  # noqa: E402
from tests.test_gpu_fuzz import random_circuit  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
nmax = int(sys.argv[3]) if len(sys.argv) > 3 else 18
bad = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, nmax + 1))
    prec = 64 if seed % 2 == 0 else 32
    kmax = int(rng.integers(1, 7))
    c = random_circuit(n, int(rng.integers(20, 120)), rng)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    p = "f64" if prec == 64 else "f32"
    sv = ts.Statevector(n, p).init_random(seed)
    re0, im0 = sv.download()
    prog = ts.Program(fused, p)
    prog.run(sv)
    dt = np.float64 if prec == 64 else np.float32
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim, threads=8)
    d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
    ok = d <= (1e-10 if prec == 64 else 1e-5)
    if not ok:
        bad += 1
        print("FAIL seed", seed, "n", n, "prec", prec, "kmax", kmax, "d", d, sorted({s["kernel"] for s in prog.steps()}))
print("done", count, "bad", bad, "env", {k: v for k, v in os.environ.items() if k.startswith("TSG_")})
