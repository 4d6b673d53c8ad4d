"""Diagonal sub-gates wider than 6 qubits (k_diag_wide).

The paper's CPU preset (FusionConfig.paper_cpu(), k_max = 7) fuses QAOA / IQP
phase layers into 7-qubit diagonals, and fuse_matrices allows unions up to 12
(gate.hpp kFusedQubitCap).  Every such gate must plan and run on the GPU
against the oracle's SPEC apply_kernel, full range and sub-ranges.
"""
import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import random_gate_matrix, random_state, to_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("k", [7, 9, 12])
def test_wide_diagonal_apply(prec, k):
    n = 15
    rng = np.random.default_rng(k)
    targets = sorted(int(q) for q in rng.choice(n, size=k, replace=False))
    m = random_gate_matrix(k, 50 + k, "diag")
    re, im = random_state(n, k)
    sv = ts.Statevector(n, "f64" if prec == 64 else "f32").upload(re, im)
    plan = ts.KernelPlan(ts.Gate(targets, m), n)
    assert plan.info()["kernel"] == "diagonal"
    T = 1 << (n - k)
    ts.apply_kernel(plan, sv, None, 0, T // 3)  # sub-range, then the rest
    ts.apply_kernel(plan, sv, None, T // 3, T)
    dt = np.float64 if prec == 64 else np.float32
    ore, oim = re.astype(dt), im.astype(dt)
    ob.apply_kernel(n, targets, m, ore, oim)
    assert ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64))) <= (1e-12 if prec == 64 else 1e-6)


def _phase_circuit(n, seed):
    """A diagonal-only circuit: cz / cp / rz / t on random qubits, like QAOA's
    and IQP's phase layers (fusion keeps every block diagonal)."""
    rng = np.random.default_rng(seed)
    c = ts.Circuit(n)
    for _ in range(6 * n):
        a, b = (int(x) for x in rng.choice(n, size=2, replace=False))
        name = ["cz", "cp", "rz", "t"][int(rng.integers(4))]
        if name == "cz":
            c.add("cz", [a, b])
        elif name == "cp":
            c.add("cp", [a, b], [float(rng.uniform(0, 3))])
        elif name == "rz":
            c.add("rz", [a], [float(rng.uniform(0, 3))])
        else:
            c.add("t", [a])
    return c


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("kmax", [8, 10, 12])
def test_wide_diagonal_blocks_in_programs(prec, kmax):
    n = 16
    fused, _ = ts.run_fusion(_phase_circuit(n, kmax), ts.FusionConfig(k_max=kmax))
    widths = [len(g.targets) for g in fused.gates()]
    assert max(widths) > 6, widths
    prog = ts.Program(fused, prec)
    sv = ts.Statevector(n, prec).init_random(4)
    re0, im0 = sv.download()
    prog.run(sv)
    dt = np.float64 if prec == "f64" else np.float32
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim, threads=4)
    d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
    assert d <= (1e-10 if prec == "f64" else 1e-5), d


def test_wide_nondiagonal_block_is_rejected_before_any_state_change():
    """Non-diagonal sub-gates above 6 qubits have no GPU kernel: Program
    creation (planning) fails with ConfigError, nothing runs."""
    n = 12
    c = ts.Circuit(n)
    c.add_matrix(list(range(7)), ob.random_unitary(7, 3))
    with pytest.raises(ts.ConfigError):
        ts.Program(c, "f64")
