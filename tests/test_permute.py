"""Qubit-permutation steps (tilesim/pass.hpp qubit_permutation, permute.cu):
a run of >= 3 consecutive gates that only permute qubits (SWAP layers, e.g.
QFT's bit reversal after fusion) is applied as one in-place involution sweep
(two sweeps when the composed permutation is not an involution).

CPU: detection and planning.  GPU: against the CPU oracle's run_circuit and
against the same program with the step disabled (TSG_NO_PERMUTE)."""
import os

import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import random_gate_matrix, to_oracle

PREC = {64: "f64", 32: "f32"}
BAR = {64: 1e-10, 32: 1e-5}


def swap_circuit(n, pairs, extra=None):
    c = ts.Circuit(n)
    if extra:
        for t, m in extra[0]:
            c.add_matrix(t, m)
    for a, b in pairs:
        c.add("swap", [a, b])
    if extra:
        for t, m in extra[1]:
            c.add_matrix(t, m)
    return c


def cswap_matrix():
    """Fredkin on sorted targets [a, b, ctl] (bit 2 = control)."""
    m = np.zeros((8, 8))
    for j in range(8):
        i = j
        if j & 4 and ((j & 1) != ((j >> 1) & 1)):
            i = j ^ 3
        m[i, j] = 1
    return m


def _kinds(c, prec="f64"):
    return [("permute" if s["is_permute"] else "pass" if s["is_pass"] else "gate", len(s["gates"]))
            for s in ts.plan_passes(c, prec)]


def test_qft30_swap_layer_is_one_step():
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", 30), ts.FusionConfig(k_max=5))
    steps = ts.plan_passes(fused, "f64")
    perm = [s for s in steps if s["is_permute"]]
    assert len(perm) == 1 and perm[0]["gates"] == list(range(106, 113))
    assert len(steps) == 7


def test_short_runs_and_controlled_swaps_stay_gates():
    n = 14
    assert all(k != "permute" for k, _ in _kinds(swap_circuit(n, [(0, 5), (7, 9)])))  # run of 2
    c = ts.Circuit(n)
    for a, b, ctl in [(0, 5, 9), (1, 6, 10), (2, 7, 11)]:
        c.add_matrix([a, b, ctl], cswap_matrix())
    assert all(k != "permute" for k, _ in _kinds(c))  # controlled: not a qubit permutation
    c = swap_circuit(n, [(0, 5), (7, 9), (3, 12)])
    assert ("permute", 3) in _kinds(c)
    os.environ["TSG_NO_PERMUTE"] = "1"
    try:
        assert all(k != "permute" for k, _ in _kinds(c))
    finally:
        os.environ.pop("TSG_NO_PERMUTE")


def _run(c, prec, psi0, env=None):
    if env:
        os.environ.update(env)
    try:
        prog = ts.Program(c, PREC[prec])
    finally:
        for k in env or {}:
            os.environ.pop(k)
    sv = ts.Statevector(c.n_qubits, PREC[prec]).upload(psi0.real.copy(), psi0.imag.copy())
    prog.run(sv)
    return sv, prog


CASES = {
    "bitrev16": (16, [(i, 15 - i) for i in range(8)]),                 # involution, every run bit moves high
    "cycle15": (15, [(i, i + 1) for i in range(14)]),                  # 15-cycle: two sweeps
    "mixed14": (14, [(0, 13), (2, 5), (5, 9), (1, 3), (12, 4), (7, 8)]),
    "low12": (12, [(0, 1), (2, 3), (1, 2), (4, 0)]),                   # permutation inside the run bits only
    "high17": (17, [(10, 16), (11, 15), (12, 14), (9, 13)]),           # no run bit moves
}


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("case", sorted(CASES))
def test_permute_step_matches_oracle(case, prec):
    n, pairs = CASES[case]
    rng = np.random.default_rng(len(pairs) * 7 + n)
    before = [([1, 6, 9], random_gate_matrix(3, 1, "dense")), ([0, n - 1], random_gate_matrix(2, 2, "dense"))]
    after = [([2, 4, n - 2], random_gate_matrix(3, 3, "dense"))]
    c = swap_circuit(n, pairs, (before, after))
    psi0 = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi0 /= np.linalg.norm(psi0)
    dt = np.float64 if prec == 64 else np.float32
    psi0 = psi0.real.astype(dt).astype(np.float64) + 1j * psi0.imag.astype(dt).astype(np.float64)
    sv, prog = _run(c, prec, psi0)
    kinds = [s["kernel"] for s in prog.steps()]
    assert any(k.startswith("k_permute") for k in kinds), kinds
    if case == "cycle15":
        assert "k_permute x2" in kinds
    ore, oim = psi0.real.astype(dt), psi0.imag.astype(dt)
    ob.run_circuit(to_oracle(c), ore, oim)
    assert ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64))) <= BAR[prec]
    ref, _ = _run(c, prec, psi0, {"TSG_NO_PERMUTE": "1"})
    # the step moves values exactly; per-gate SWAP kernels may round (3M product)
    assert ts.compare_states(sv, ref) <= (1e-14 if prec == 64 else 1e-6)


@pytest.mark.gpu
def test_qft_with_permute_step_analytic():
    """QFT|x> (closed form) through passes + the bit-reversal permutation step."""
    n, x = 20, 0x5A3C7
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", n), ts.FusionConfig(k_max=5))
    prog = ts.Program(fused, "f64")
    assert any(s["kernel"].startswith("k_permute") for s in prog.steps())
    sv = ts.Statevector(n, "f64").init_basis(x)
    prog.run(sv)
    y = np.arange(1 << n)
    want = np.exp(2j * np.pi * ((x * y) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
    assert np.abs(sv.amplitudes() - want).max() <= 1e-10
