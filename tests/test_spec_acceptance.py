"""SPEC acceptance criteria 1-9 at desk scale, on the CPU
oracle (kernel/sim) with fusion plans from both the oracle and the product."""
import itertools
import time

import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import circuits_equal, random_state
from tests.test_host_surface import COST_MODEL

NAMED = [("h", 1, 0), ("x", 1, 0), ("y", 1, 0), ("z", 1, 0), ("s", 1, 0), ("t", 1, 0), ("rx", 1, 1), ("ry", 1, 1),
         ("rz", 1, 1), ("u3", 1, 3), ("cx", 2, 0), ("cz", 2, 0), ("cp", 2, 1), ("swap", 2, 0), ("ccx", 3, 0)]


def random_circuit(rng, n, n_gates):
    c = ob.Circuit(n)
    for _ in range(n_gates):
        if rng.random() < 0.2:
            k = int(rng.integers(1, min(3, n) + 1))
            q = rng.choice(n, k, replace=False).tolist()
            c.add_matrix(q, ob.random_unitary(k, int(rng.integers(1 << 30))))
            continue
        name, arity, npar = NAMED[int(rng.integers(len(NAMED)))]
        if arity > n:
            continue
        c.add(name, rng.choice(n, arity, replace=False).tolist(), rng.uniform(-3, 3, npar).tolist())
    return c


def test_c1_oracle_equivalence():
    """200 random circuits x fusion modes x s in {0..3} x threads in {1, 4}: fused
    specialised run == dense reference_apply on the unfused circuit."""
    rng = np.random.default_rng(1)
    cm = ob.CostModel(COST_MODEL)
    t0 = time.time()
    worst = 0.0
    for i in range(200):
        n = int(rng.integers(2, 9))
        c = random_circuit(rng, n, int(rng.integers(1, 61)))
        re, im = random_state(n, i)
        rre, rim = re.copy(), im.copy()
        ob.reference_run(c, rre, rim)
        mode = ("none", "size", "adaptive")[i % 3]
        f, _ = ob.run_fusion(c, mode, k_max=min(4, n), cost_model=cm if mode == "adaptive" else None)
        kmax = max([len(t) for t, _, _ in f.gates()] or [1])
        s = max(0, min(i % 4, n - kmax))  # plan_kernel rejects k + s > n
        fre, fim = re.copy(), im.copy()
        ob.run_circuit(f, fre, fim, threads=1 + 3 * (i % 2), s=s)
        worst = max(worst, ob.compare_states(fre, fim, rre, rim))
    assert worst <= 1e-12, worst
    assert time.time() - t0 < 120


def test_c2_op_count_law():
    for k in range(1, 7):
        _, cnt = ob.profile(ob.random_unitary(k, 7 + k), 1e-8, 0.0)
        assert cnt["op_count"] == 2 ** (2 * k + 2)
        g = ts.Gate(list(range(k)), ob.random_unitary(k, 7 + k))
        assert ts.KernelPlan(g, k, one_tol=0.0).info()["op_count"] == 2 ** (2 * k + 2)


def test_c3_index_completeness():
    for n in range(1, 13):
        full = np.arange(1 << n, dtype=np.uint64)
        for k in range(1, min(4, n) + 1):
            for t in itertools.combinations(range(n), k):
                for s in range(4):
                    if k + s >= n and not (k + s == n):
                        continue
                    if k + s > n:
                        continue
                    idx = ob.enumerate_indices(list(t), s, n)
                    assert np.array_equal(np.sort(idx), full), (n, t, s)


def test_c4_qft16_analytic_paper_cpu_preset():
    n = 16
    cm = ob.CostModel(COST_MODEL)
    f, _ = ob.run_fusion(ob.gen_benchmark("qft", n), "adaptive", k_max=7, max_op_count=4096, cost_model=cm)
    re, im = ob.zero_state(n)
    t0 = time.time()
    ob.run_circuit(f, re, im, threads=4)
    mod = np.sqrt(re * re + im * im)
    assert np.abs(mod - 2 ** -8).max() <= 1e-12
    assert time.time() - t0 < 10
    # the product plans the same fused circuit bit-for-bit
    pf, _ = ts.run_fusion(ts.gen_benchmark("qft", n),
                          ts.FusionConfig(k_max=7, max_op_count=4096, mode="adaptive"), ts.CostModel(COST_MODEL))
    circuits_equal(pf, f)


@pytest.mark.parametrize("kind,depth", [("qft", 1), ("iqp", 6), ("hes", 6)])
def test_c5_fusion_ablation_direction(kind, depth):
    n = 18
    c = ob.gen_benchmark(kind, n, depth, 3)
    cm = ob.CostModel(COST_MODEL)
    fs, sts = ob.run_fusion(c, "size", k_max=5)
    fa, sta = ob.run_fusion(c, "adaptive", k_max=7, max_op_count=4096, cost_model=cm)
    assert sta["total_op_count"] <= sts["total_op_count"] * 1.0 + 1e-9 or sta["fused_block_count"] <= sts[
        "fused_block_count"]
    re, im = ob.zero_state(n)
    t_none = ob.run_circuit(c, re.copy(), im.copy(), threads=4)["execution_s"]
    t_size = ob.run_circuit(fs, re.copy(), im.copy(), threads=4)["execution_s"]
    assert t_size <= 0.5 * t_none, (t_size, t_none)


def test_c6_fixed_point_and_conservation():
    rng = np.random.default_rng(6)
    for i in range(100):
        n = int(rng.integers(2, 8))
        c = random_circuit(rng, n, int(rng.integers(1, 40)))
        f, st = ob.run_fusion(c, "size", k_max=min(4, n))
        again, st2 = ob.run_fusion(f, "size", k_max=min(4, n), agglomerative=False)
        # a fused circuit is a fixed point at the same k unless two blocks still fit together
        assert st2["fused_block_count"] <= st["fused_block_count"]
        for t, m, _ in f.gates():
            assert ob.is_unitary(m, 1e-9)
        re, im = random_state(n, i)
        a = (re.copy(), im.copy())
        b = (re.copy(), im.copy())
        ob.reference_run(c, *a)
        ob.reference_run(f, *b)
        assert ob.compare_states(*a, *b) <= 1e-12


def test_c7_thread_invariance():
    n = 16
    f, _ = ob.run_fusion(ob.gen_benchmark("rqc", n, 10, 7), "size", k_max=5)
    re, im = random_state(n, 7)
    outs = []
    for threads in (1, 2, 4, 8):
        r, i = re.copy(), im.copy()
        ob.run_circuit(f, r, i, threads=threads)
        outs.append((r, i))
    for r, i in outs[1:]:
        assert ob.compare_states(r, i, *outs[0]) <= 1e-13


def test_c8_front_end_fraction():
    n = 22
    t0 = time.perf_counter()
    c = ts.gen_benchmark("rqc", n, 12, 1)
    f, st = ts.run_fusion(c, ts.FusionConfig(k_max=5))
    front = time.perf_counter() - t0
    o = ob.Circuit(n)
    for g in f.gates():
        o.add_matrix(g.targets, g.matrix)
    re, im = ob.zero_state(n)
    back = ob.run_circuit(o, re, im, threads=8)["execution_s"]
    assert front / (front + back) < 0.2


def test_c9_cost_model_round_trip_and_caps():
    cm = ts.CostModel(COST_MODEL)
    cm2 = ts.CostModel(cm.serialize())
    c = ts.gen_benchmark("ala", 10, 6, 2)
    f, _ = ts.run_fusion(c, ts.FusionConfig(k_max=6, max_op_count=1024, mode="adaptive"), cm2)
    for g in f.gates():
        assert g.k <= 6
        if not g.name:
            assert ts.KernelPlan(g, 10).info()["op_count"] <= 1024
