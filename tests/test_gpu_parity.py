"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): complex128 max |dpsi| <= 1e-10, complex64
<= 1e-5, fidelity >= 1 - 1e-9, on the SAME kernel plan (same tolerances and
scalar kinds) as the oracle's SPEC apply_kernel.
"""
import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import random_gate_matrix, random_state, to_oracle

pytestmark = pytest.mark.gpu

TOL = {64: 1e-12, 32: 1e-5}
PREC = {64: "f64", 32: "f32"}

TARGET_SETS = {
    1: [[0], [1], [3], [9]],
    2: [[0, 1], [0, 5], [2, 7], [6, 11]],
    3: [[0, 1, 2], [0, 3, 8], [4, 9, 12], [1, 2, 10]],
    4: [[0, 1, 2, 3], [0, 2, 6, 11], [5, 7, 9, 12]],
    5: [[0, 1, 2, 3, 4], [1, 4, 6, 9, 12], [3, 5, 7, 8, 13]],
    6: [[0, 1, 2, 3, 4, 5], [0, 2, 5, 7, 10, 13], [6, 7, 8, 9, 10, 11]],
}


def _gpu_apply(n, targets, m, re, im, prec, override=None, t_begin=0, t_end=None, runtime=False):
    sv = ts.Statevector(n, PREC[prec]).upload(re, im)
    plan = ts.KernelPlan(ts.Gate(list(targets), m), n, runtime_matrix=runtime)
    ts.apply_kernel(plan, sv, override, t_begin, t_end)
    return sv, plan


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("kind", ["dense", "perm", "diag", "controlled"])
def test_apply_matches_oracle(prec, k, kind):
    n = 14
    ts.default_context()
    for i, targets in enumerate(TARGET_SETS[k]):
        m = random_gate_matrix(k, 100 * k + i, kind)
        dt = np.float64 if prec == 64 else np.float32
        re, im = random_state(n, 7 + i, dt)
        sv, plan = _gpu_apply(n, targets, m, re.astype(np.float64), im.astype(np.float64), prec)
        ore, oim = re.copy(), im.copy()
        ob.apply_kernel(n, targets, m, ore, oim)  # SPEC apply_kernel, same precision
        d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
        assert d <= TOL[prec], (k, kind, targets, plan.info(), d)


@pytest.mark.parametrize("prec", [64, 32])
def test_named_gate_classes(prec):
    """Control peeling and kernel-class selection on the named gates."""
    n = 12
    cases = [("cx", [2, 7], "direct", 1, 1), ("cx", [7, 2], "direct", 1, 1), ("cz", [0, 5], "diagonal", 0, 2),
             ("cp", [3, 4], "diagonal", 0, 2), ("rz", [5], "diagonal", 1, 0), ("t", [0], "diagonal", 0, 1),
             ("h", [0], "direct", 1, 0), ("ccx", [1, 4, 9], "direct", 1, 2), ("swap", [2, 10], "direct", 2, 0),
             ("x", [11], "direct", 1, 0), ("y", [0], "direct", 1, 0)]
    for name, qubits, klass, sub_k, ctrl in cases:
        params = [0.7] if name in ("cp", "rz") else []
        g = ts.make_named_gate(name, params, qubits)
        re, im = random_state(n, 3)
        sv, plan = _gpu_apply(n, g.targets, g.matrix, re, im, prec)
        info = plan.info()
        assert (info["kernel"], info["sub_k"], info["n_controls"]) == (klass, sub_k, ctrl), (name, info)
        ore = re.astype(np.float64 if prec == 64 else np.float32)
        oim = im.astype(ore.dtype)
        ob.apply_kernel(n, g.targets, g.matrix, ore, oim)
        assert ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64))) <= TOL[prec], name


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("k,targets", [(1, [0]), (2, [1, 6]), (3, [0, 4, 9]), (5, [0, 1, 3, 8, 10]),
                                       (6, [2, 3, 4, 5, 6, 7])])
def test_subrange_partition(prec, k, targets):
    """Disjoint [t_begin, t_end) calls compose to the full application."""
    n = 13
    m = random_gate_matrix(k, 5, "dense")
    re, im = random_state(n, 11)
    full, _ = _gpu_apply(n, targets, m, re, im, prec)
    sv = ts.Statevector(n, PREC[prec]).upload(re, im)
    plan = ts.KernelPlan(ts.Gate(targets, m), n)
    T = 1 << (n - k)
    cuts = sorted({0, T, T // 3, T // 2 + 1, (7 * T) // 8})
    for a, b in zip(cuts[:-1], cuts[1:]):
        ts.apply_kernel(plan, sv, None, a, b)
    assert ts.compare_states(sv, full) <= TOL[prec] / 10


def test_runtime_matrix_override():
    n = 12
    targets = [1, 5]
    m = random_gate_matrix(2, 1, "dense")
    m2 = random_gate_matrix(2, 2, "dense")
    re, im = random_state(n, 4)
    sv, plan = _gpu_apply(n, targets, m, re, im, 64, override=m2, runtime=True)
    ore, oim = re.copy(), im.copy()
    ob.apply_kernel(n, targets, m, ore, oim, override=m2)
    assert ts.compare_states(sv, (ore, oim)) <= 1e-12
    # an override whose sparsity differs from the plan is a SimError
    with pytest.raises(ts.SimError):
        ts.apply_kernel(plan, sv, np.eye(4))
    # a baked plan refuses overrides
    baked = ts.KernelPlan(ts.Gate(targets, m), n)
    with pytest.raises(ts.SimError):
        ts.apply_kernel(baked, sv, m2)


@pytest.mark.parametrize("kind,n,depth,prec,kmax", [
    ("qft", 16, 1, 64, 5), ("rqc", 16, 12, 64, 5), ("ala", 14, 6, 64, 4), ("qvc", 14, 4, 64, 5),
    ("iqp", 16, 4, 64, 5), ("hes", 16, 4, 64, 5), ("qaoa", 16, 4, 32, 6), ("qaoa", 16, 4, 32, 3),
    ("rqc", 14, 10, 32, 6), ("qft", 12, 1, 64, 6),
])
def test_fused_circuit_matches_oracle(kind, n, depth, prec, kmax):
    c = ts.gen_benchmark(kind, n, depth, 42)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    sv = ts.Statevector(n, PREC[prec]).init_random(1)
    re0, im0 = sv.download()
    rep = ts.run_circuit(fused, sv)
    assert rep["gates"] == len(fused)
    dt = np.float64 if prec == 64 else np.float32
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim, threads=4)
    d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
    bar = 1e-10 if prec == 64 else 1e-5
    assert d <= bar, d
    # against the unfused dense oracle in fp64 as well (fidelity bar)
    rre, rim = re0.copy(), im0.copy()
    ob.reference_run(to_oracle(c), rre, rim)
    psi = sv.amplitudes()
    ref = rre + 1j * rim
    # normalised fidelity (the north star's bar for both precisions); the
    # norm itself is checked by the max |dpsi| bar above
    fid = abs(np.vdot(ref, psi)) ** 2 / (np.vdot(ref, ref).real * np.vdot(psi, psi).real)
    assert fid >= 1 - 1e-9, 1 - fid


def test_qft_analytic_basis_state():
    """QFT|x> = sum_y e^{2 pi i x y / 2^n} |y> / 2^{n/2} (SURVEY.md §8c extra oracle 1)."""
    n, x = 20, 0x5A5A5
    c = ts.gen_benchmark("qft", n)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=5))
    sv = ts.Statevector(n, "f64").init_basis(x)
    ts.run_circuit(fused, sv)
    y = np.arange(1 << n)
    want = np.exp(2j * np.pi * ((x * y) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
    assert np.abs(sv.amplitudes() - want).max() <= 1e-10


def test_norm_compare_init():
    sv = ts.Statevector(16, "f64").init_random(9)
    re, im = sv.download()
    assert abs(sv.norm() - 1.0) < 1e-12
    assert abs(sv.norm() - np.sqrt((re * re + im * im).sum())) < 1e-13
    other = ts.Statevector(16, "f64").init_random(9)
    assert ts.compare_states(sv, other) == 0.0
    z = ts.Statevector(16, "f32").init_zero()
    zr, zi = z.download()
    assert zr[0] == 1.0 and zr[1:].sum() == 0 and zi.sum() == 0
    assert abs(ts.compare_states(z, (re, im)) - np.sqrt(((zr - re) ** 2 + (zi - im) ** 2).max())) < 1e-6
    assert abs(ts.overlap(sv, other) - 1.0) < 1e-12


def test_program_graph_and_profile():
    c = ts.gen_benchmark("rqc", 18, 8, 3)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=4))
    prog = ts.Program(fused, "f64")
    a = ts.Statevector(18, "f64").init_random(2)
    b = ts.Statevector(18, "f64").copy_from(a)
    r1 = prog.run(a, use_graph=True)
    secs, r2 = prog.run_profiled(b)
    assert ts.compare_states(a, b) == 0.0
    assert r1["launches"] == r2["launches"] and len(secs) == len(fused) and (secs >= 0).all()
    prog.run(a, use_graph=True)  # cached graph replay
    prog.run(b, use_graph=False)
    assert ts.compare_states(a, b) == 0.0


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("n,kmax", [(1, 1), (2, 2), (3, 3), (4, 4), (5, 5), (6, 5), (7, 6), (8, 5), (10, 5),
                                    (10, 6), (12, 5), (13, 6)])
def test_small_states_every_kernel_path(n, kmax, prec):
    """States smaller than a tile pass / a tensor-core tile: the executor must
    pick kernels that fit (per-gate launches, smaller products) and still match
    the oracle; random fused circuits with 1..kmax-qubit blocks."""
    rng = np.random.default_rng(n * 10 + prec)
    c = ts.Circuit(n)
    for i in range(40):
        k = int(rng.integers(1, min(5, n) + 1))
        t = sorted(int(q) for q in rng.choice(n, size=k, replace=False))
        kind = ["dense", "perm", "diag", "controlled"][i % 4] if k > 1 else "dense"
        c.add_matrix(t, random_gate_matrix(k, 700 + i, kind))
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    sv = ts.Statevector(n, PREC[prec]).init_random(2)
    re0, im0 = sv.download()
    ts.run_circuit(fused, sv)
    dt = np.float64 if prec == 64 else np.float32
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim)
    assert ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64))) <= (1e-10 if prec == 64 else 1e-5)


@pytest.mark.parametrize("targets", [[0, 1, 2, 3, 4, 5], [1, 3, 5, 8, 12, 17], [14, 15, 16, 17, 18, 19],
                                     [0, 6, 7, 11, 18, 19]])
def test_dmma6_complex128(targets):
    """Dense and controlled complex128 6-qubit products on the FP64 tensor
    pipe (k_stream_dmma<ks=6>) against the oracle's apply_kernel."""
    n = 20
    for kind in ("dense", "controlled"):
        m = random_gate_matrix(6, sum(targets) + len(kind), kind)
        re, im = random_state(n, 11)
        sv, plan = _gpu_apply(n, targets, m, re, im, 64)
        if kind == "dense":
            c = ts.Circuit(n)
            c.add_matrix(targets, m)
            assert ts.Program(c, "f64").steps()[0]["kernel"] == "k_stream_dmma<ks=6>"
        ore, oim = re.copy(), im.copy()
        ob.apply_kernel(n, targets, m, ore, oim)
        d = ts.compare_states(sv, (ore, oim))
        assert d <= 1e-12, (kind, targets, plan.info(), d)


def _tile_sparse_matrix(k, seed, density=0.5):
    """A random (non-unitary) matrix whose 8x4 DMMA tiles (natural order) are
    zero with probability 1 - density."""
    rng = np.random.default_rng(seed)
    d = 1 << k
    m = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    tiles = [(rb, kb) for rb in range(d // 8) for kb in range(d // 4)][1:]  # tile (0, 0) stays dense
    zero = [t for t in tiles if rng.uniform() > density] or tiles[-1:]    # at least one zero tile
    for rb, kb in zero:
        m[8 * rb:8 * rb + 8, 4 * kb:4 * kb + 4] = 0
    return m / np.sqrt(d)


@pytest.mark.parametrize("ks", [3, 4, 5])
def test_dmma_jit_zero_tiles(ks, monkeypatch):
    """Standalone complex128 DMMA products JIT-compiled with their zero tiles
    compiled out: bit-identical to the generic kernels (dense or runtime
    predicates), and against the oracle."""
    monkeypatch.setenv("TSG_PASS_JIT_MIN_N", "1")
    monkeypatch.setenv("TSG_NO_PASS", "1")
    monkeypatch.setenv("TSG_NO_BLOCK_SPLIT", "1")
    n = 16
    rng = np.random.default_rng(ks)
    c = ts.Circuit(n)
    for i, density in enumerate((0.25, 0.5, 0.75, 0.45, 0.55, 0.5)):
        t = sorted(int(q) for q in rng.choice(n, size=ks, replace=False)) if i else list(range(ks))
        c.add_matrix(t, _tile_sparse_matrix(ks, 10 * ks + i, density))
    pj = ts.Program(c, "f64")
    assert pj.jit_kernels()["gates"] >= 2, pj.jit_kernels()  # (the mid-density ones: dmma_jit_spec)
    monkeypatch.setenv("TSG_DMMA_JIT", "0")
    p0 = ts.Program(c, "f64")
    assert p0.jit_kernels()["gates"] == 0
    a = ts.Statevector(n, "f64").init_random(3)
    b = ts.Statevector(n, "f64").copy_from(a)
    re0, im0 = a.download()
    pj.run(a)
    p0.run(b)
    assert ts.compare_states(a, b) == 0.0
    ore, oim = re0.copy(), im0.copy()
    ob.run_circuit(to_oracle(c), ore, oim, threads=4)
    assert ts.compare_states(a, (ore, oim)) <= 1e-12


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_state_gather(prec):
    """tsg_state_gather: amplitudes at arbitrary indices equal the downloaded state's."""
    n = 14
    sv = ts.Statevector(n, prec).init_random(5)
    re, im = sv.download()
    idx = np.random.default_rng(1).integers(0, 1 << n, size=77)
    gr, gi = sv.gather(idx)
    assert np.array_equal(gr, re[idx]) and np.array_equal(gi, im[idx])
    with pytest.raises(ts.TilesimError):
        sv.gather([1 << n])
