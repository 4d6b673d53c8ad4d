"""Tile passes (tilesim/pass.hpp, k_pass): several fused gates per HBM sweep.

CPU tests check the planner (coverage, order, tile-qubit budget, which gates
may join a pass).  GPU tests check k_pass through the C ABI against the CPU
oracle's SPEC run_circuit (same kernel plans) and
against the same program with passes disabled.
"""
import os

import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import block_gate, random_gate_matrix, to_oracle

PREC = {64: "f64", 32: "f32"}
BAR = {64: 1e-10, 32: 1e-5}
GEOM = {64: (11, 5, 4), 32: (12, 6, 5)}  # tile_log2, run_log2, widest GEN sub-gate


def mixed_circuit(n: int, n_gates: int, seed: int) -> ts.Circuit:
    """Named and matrix gates on random qubits: controls and diagonal targets
    land inside and outside any tile, low and high."""
    rng = np.random.default_rng(seed)
    c = ts.Circuit(n)
    for i in range(n_gates):
        r = rng.integers(0, 10)
        q = [int(x) for x in rng.choice(n, size=3, replace=False)]
        if r == 0:
            c.add("cx", q[:2])
        elif r == 1:
            c.add("ccx", q)
        elif r == 2:
            c.add("cp", q[:2], [float(rng.uniform(0, 6.28))])
        elif r == 3:
            c.add("h", q[:1])
        elif r == 4:
            c.add("rz", q[:1], [float(rng.uniform(0, 6.28))])
        elif r == 5:
            c.add("u3", q[:1], [float(x) for x in rng.uniform(0, 6.28, 3)])
        elif r == 6:
            c.add("swap", q[:2])
        else:
            k = int(rng.integers(1, 4))
            kind = ["dense", "perm", "diag", "controlled"][int(rng.integers(0, 4))]
            c.add_matrix(sorted(q[:k]), random_gate_matrix(k, seed * 1000 + i, kind))
    return c


def mixed_qubits(gate, zero_tol=1e-8):
    """Qubits a gate mixes: some entry that is not Zero (SPEC classify) links
    rows and columns differing in that qubit (tilesim::mixed_bits)."""
    m = np.asarray(gate.matrix)
    nz = (np.abs(m.real) > zero_tol) | (np.abs(m.imag) > zero_tol)
    r, c = np.nonzero(nz)
    x = np.bitwise_or.reduce(r ^ c) if len(r) else 0
    return [q for b, q in enumerate(gate.targets) if (x >> b) & 1]


def assert_reorder_commutes(fused, order):
    """The lookahead planner may run a gate before earlier ones: every such
    inverted pair must commute (each shared qubit a block qubit of both)."""
    qs = {g: (set(fused.gate(g).targets), set(mixed_qubits(fused.gate(g)))) for g in order}
    pos = {g: i for i, g in enumerate(order)}
    for a in order:
        for b in order:
            if a < b and pos[b] < pos[a]:
                (qa, ma), (qb, mb) = qs[a], qs[b]
                assert not ((qa & qb) & (ma | mb)), (a, b, qa & qb, ma, mb)


# ----------------------------------------------------------------- planner
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("kind,n,depth,kmax", [("qft", 30, 1, 5), ("rqc", 24, 12, 4), ("qaoa", 26, 4, 4),
                                               ("hes", 20, 6, 5), ("iqp", 22, 4, 3), ("mixed", 20, 300, 3)])
def test_plan_passes_properties(prec, kind, n, depth, kmax):
    c = mixed_circuit(n, depth, 5) if kind == "mixed" else ts.gen_benchmark(kind, n, depth, 42)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    M, L, gen_max = GEOM[prec]
    steps = ts.plan_passes(fused, PREC[prec])
    seen = [g for s in steps for g in s["gates"]]
    assert len(seen) == len(set(seen)), "each gate once"
    assert_reorder_commutes(fused, seen)
    for s in steps:
        if s["is_permute"]:  # a run of qubit permutations (tests/test_permute.py)
            assert len(s["gates"]) >= 3 and s["high"] == []
            continue
        if not s["is_pass"]:
            assert len(s["gates"]) == 1 and s["high"] == []
            continue
        assert len(s["gates"]) >= 2
        assert len(s["high"]) == M - L and s["high"] == sorted(set(s["high"]))
        assert all(L <= h < n for h in s["high"])
        tile = set(range(L)) | set(s["high"])
        for g in s["gates"]:
            p = ts.plan_kernel(fused.gate(g), n).info()
            assert p["kernel"] != "identity"
            if p["kernel"] != "diagonal":
                mixed = mixed_qubits(fused.gate(g))
                assert 1 <= len(mixed) <= gen_max
                assert set(mixed) <= tile, (g, mixed, tile)  # every qubit the gate mixes is a tile qubit
    # every non-identity gate is launched exactly once
    for gi in range(len(fused)):
        if ts.plan_kernel(fused.gate(gi), n).info()["kernel"] != "identity":
            assert gi in seen


def test_plan_passes_qft30_sweeps():
    """QFT-30 (k<=5): 113 fused gates become a handful of HBM sweeps."""
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", 30), ts.FusionConfig(k_max=5))
    steps = ts.plan_passes(fused, "f64")
    assert len(fused) == 113
    assert len(steps) <= 16
    assert sum(len(s["gates"]) for s in steps if s["is_pass"]) >= 100


def test_plan_passes_small_state_has_no_pass():
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", 10), ts.FusionConfig(k_max=3))
    assert not any(s["is_pass"] for s in ts.plan_passes(fused, "f64"))


# --------------------------------------------------------------------- GPU
def _run_program(fused, prec, re0, im0, no_pass=False, force=False):
    if no_pass:
        os.environ["TSG_NO_PASS"] = "1"
    if force:
        os.environ["TSG_PASS_FORCE"] = "1"
    try:
        prog = ts.Program(fused, PREC[prec])
    finally:
        os.environ.pop("TSG_NO_PASS", None)
        os.environ.pop("TSG_PASS_FORCE", None)
    sv = ts.Statevector(fused.n_qubits, PREC[prec]).upload(re0, im0)
    prog.run(sv)
    return sv, prog


@pytest.mark.gpu
@pytest.mark.parametrize("force", [True, False])
@pytest.mark.parametrize("kind,n,depth,prec,kmax", [
    ("qft", 16, 1, 64, 5), ("qft", 17, 1, 32, 5), ("rqc", 15, 10, 64, 4), ("rqc", 16, 10, 32, 5),
    ("qaoa", 16, 4, 32, 4), ("qaoa", 14, 4, 64, 3), ("hes", 16, 6, 64, 5), ("iqp", 15, 4, 64, 3),
    ("ala", 14, 4, 64, 2), ("qvc", 15, 4, 32, 4), ("mixed", 15, 400, 64, 3), ("mixed", 16, 400, 32, 4),
    ("mixed", 13, 300, 32, 2), ("mixed", 12, 300, 64, 1), ("mixed", 11, 200, 64, 2), ("mixed", 12, 200, 32, 3),
])
def test_pass_program_matches_oracle(kind, n, depth, prec, kmax, force):
    """force: every eligible gate runs inside a pass (all op kinds, any size);
    otherwise the B200 cost model decides which gates join passes."""
    c = mixed_circuit(n, depth, 11) if kind == "mixed" else ts.gen_benchmark(kind, n, depth, 42)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    rng = np.random.default_rng(3)
    re0 = rng.standard_normal(1 << n)
    im0 = rng.standard_normal(1 << n)
    s = np.sqrt((re0 ** 2 + im0 ** 2).sum())
    re0, im0 = re0 / s, im0 / s
    dt = np.float64 if prec == 64 else np.float32
    re0, im0 = re0.astype(dt).astype(np.float64), im0.astype(dt).astype(np.float64)
    sv, prog = _run_program(fused, prec, re0, im0, force=force)
    steps = prog.steps()
    if force:
        assert any(st["kind"] == "pass" for st in steps), "the case must exercise k_pass"
        os.environ["TSG_PASS_FORCE"] = "1"
    try:
        planned = ts.plan_passes(fused, PREC[prec])
    finally:
        os.environ.pop("TSG_PASS_FORCE", None)
    assert [st["kind"] == "pass" for st in steps] == [p["is_pass"] for p in planned]
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim, threads=4)
    d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
    assert d <= BAR[prec], d
    ref, _ = _run_program(fused, prec, re0, im0, no_pass=True)
    assert ts.compare_states(sv, ref) <= (1e-12 if prec == 64 else 2e-6)


@pytest.mark.gpu
def test_pass_qft_analytic_basis_state():
    """QFT|x> closed form through passes with out-of-tile diagonal bits."""
    n, x = 22, 0x2A5A5
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", n), ts.FusionConfig(k_max=5))
    prog = ts.Program(fused, "f64")
    assert sum(st["kind"] == "pass" for st in prog.steps()) >= 3
    sv = ts.Statevector(n, "f64").init_basis(x)
    prog.run(sv)
    y = np.arange(1 << n)
    want = np.exp(2j * np.pi * ((x * y) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
    assert np.abs(sv.amplitudes() - want).max() <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("mixed,block", [
    ([3, 11, 15], [9, 13]), ([3, 11, 15], []), ([11, 15], [9]), ([3], [9, 13]), ([2, 4], []), ([7, 8, 9], [12]),
    ([0, 1], [5, 14]), ([6], []), ([5, 6, 7, 8], []), ([1, 2, 3, 4], [10]), ([4, 5, 6, 7, 8], []),
])
def test_forced_single_op_pass(prec, mixed, block):
    """One block-structured gate (+ a phase) forced into a tile pass -- register
    or shared-memory op depending on its width and the layout -- against the
    same gate without passes and against the oracle."""
    n = 16
    targets, m = block_gate(mixed, block, sum(mixed) * 31 + len(block))
    c = ts.Circuit(n)
    c.add_matrix(targets, m)
    c.add_matrix([0], np.diag([1, np.exp(0.3j)]))
    rng = np.random.default_rng(1)
    re0, im0 = rng.standard_normal(1 << n), rng.standard_normal(1 << n)
    s = np.sqrt((re0 ** 2 + im0 ** 2).sum())
    dt = np.float64 if prec == 64 else np.float32
    re0, im0 = (re0 / s).astype(dt).astype(np.float64), (im0 / s).astype(dt).astype(np.float64)
    sv, prog = _run_program(c, prec, re0, im0, force=True)
    in_pass = len(mixed) <= GEOM[prec][2]  # wider sub-gates always run on their own kernel
    assert (prog.steps()[0]["kind"] == "pass") == in_pass
    ref, _ = _run_program(c, prec, re0, im0, no_pass=True)
    assert ts.compare_states(sv, ref) <= (1e-12 if prec == 64 else 2e-6)
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(c), ore, oim)
    assert ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64))) <= BAR[prec]


def test_c64_low_target_runs_join_passes():
    """complex64 4-qubit gates on a low target run from qubit 0 would fall back
    to the FP64-widened DMMA product (~2.8 sweeps): the planner prices them so
    and puts them into passes (HES-24 c64, k <= 5)."""
    fused, _ = ts.run_fusion(ts.gen_benchmark("hes", 24, 6, 42), ts.FusionConfig(k_max=5))
    steps = ts.plan_passes(fused, "f32")
    in_pass = {g for s in steps if s["is_pass"] for g in s["gates"]}
    low = [i for i in range(len(fused))
           if list(fused.gate(i).targets)[:2] == [0, 1] and len(fused.gate(i).targets) >= 4
           and ts.plan_kernel(fused.gate(i), 24).info()["kernel"] != "diagonal"]
    assert low, "the case must contain low-run gates"
    assert all(i in in_pass for i in low), (low, in_pass)
