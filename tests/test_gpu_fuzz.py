"""Randomised end-to-end parity: random circuits (named gates, SWAP layers,
dense / permutation / diagonal / controlled matrices on random qubits) at
random sizes, fusion widths and precisions, through Program (tile passes,
permutation steps, tensor-core products, block splits) against the CPU
oracle's SPEC run_circuit on the same fused circuit."""
import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import random_gate_matrix, to_oracle

pytestmark = pytest.mark.gpu


def random_circuit(n, n_gates, rng):
    c = ts.Circuit(n)
    for i in range(n_gates):
        r = int(rng.integers(0, 12))
        q = [int(x) for x in rng.choice(n, size=min(n, 6), replace=False)]
        if r == 0:
            c.add("h", q[:1])
        elif r == 1:
            c.add("cx", q[:2])
        elif r == 2:
            c.add("cp", q[:2], [float(rng.uniform(0, 6.3))])
        elif r == 3:
            for _ in range(int(rng.integers(3, 6))):  # a SWAP layer
                a, b = (int(x) for x in rng.choice(n, size=2, replace=False))
                c.add("swap", [a, b])
        elif r == 4:
            c.add("rz", q[:1], [float(rng.uniform(0, 6.3))])
        else:
            k = int(rng.integers(1, 6))
            kind = ["dense", "perm", "diag", "controlled"][int(rng.integers(0, 4))]
            c.add_matrix(sorted(q[:k]), random_gate_matrix(k, int(rng.integers(1 << 30)), kind))
    return c


@pytest.mark.parametrize("seed", range(16))
def test_random_circuits_match_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(9, 17))
    prec = 64 if seed % 2 == 0 else 32
    kmax = int(rng.integers(1, 7))
    c = random_circuit(n, int(rng.integers(30, 90)), rng)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    p = "f64" if prec == 64 else "f32"
    sv = ts.Statevector(n, p).init_random(seed)
    re0, im0 = sv.download()
    prog = ts.Program(fused, p)
    prog.run(sv)
    dt = np.float64 if prec == 64 else np.float32
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim, threads=4)
    d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
    kernels = sorted({s["kernel"] for s in prog.steps()})
    assert d <= (1e-10 if prec == 64 else 1e-5), (n, prec, kmax, d, kernels)
