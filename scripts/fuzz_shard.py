"""Randomised parity of the sharded executor (virtual shards on one GPU):
random circuits (tests/test_gpu_fuzz.py) over 2^g shards vs the CPU oracle.
usage: fuzz_shard.py FIRST_SEED COUNT"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402
from oracle import binding as ob  # noqa: E402
from tests._util import random_state, to_oracle  # noqa: E402
from tests.test_gpu_fuzz import random_circuit  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(10, 17))
    g = int(rng.integers(1, 4))
    prec = "f64" if seed % 2 == 0 else "f32"
    kmax = int(rng.integers(1, 6))
    c = random_circuit(n, int(rng.integers(20, 80)), rng)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    plan = ts.ShardPlan(fused, g)
    re, im = random_state(n, seed)
    if prec == "f32":
        re, im = re.astype(np.float32).astype(np.float64), im.astype(np.float32).astype(np.float64)
    got_re, got_im, rep = ts.vshard_run(plan, re, im, prec)
    dt = np.float64 if prec == "f64" else np.float32
    ore, oim = re.astype(dt), im.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim, threads=8)
    d = np.abs((got_re - ore) + 1j * (got_im - oim)).max()
    if d > (1e-10 if prec == "f64" else 1e-5):
        bad += 1
        print("FAIL seed", seed, "n", n, "g", g, prec, "kmax", kmax, "d", d, plan.info())
print("done", count, "bad", bad)
