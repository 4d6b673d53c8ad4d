"""Sharded execution on the device: 2^g virtual shards on one B200 (the
single-GPU emulation of the distributed path) against the
unsharded device run and the CPU oracle; the NCCL executor at world size 1."""
import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import random_state, to_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,depth,kmax,prec", [("qft", 14, 1, 5, "f64"), ("rqc", 14, 8, 5, "f64"),
                                                    ("qaoa", 14, 3, 4, "f32"), ("hes", 13, 3, 4, "f64"),
                                                    ("ala", 12, 4, 3, "f64")])
@pytest.mark.parametrize("g", [1, 2, 3])
def test_vshard_matches_unsharded(kind, n, depth, kmax, prec, g):
    c = ts.gen_benchmark(kind, n, depth, 5)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    plan = ts.ShardPlan(fused, g)
    re, im = random_state(n, 3)
    got_re, got_im, rep = ts.vshard_run(plan, re, im, prec)
    sv = ts.Statevector(n, prec).upload(re, im)
    ts.run_circuit(fused, sv)
    bar = 1e-10 if prec == "f64" else 1e-5
    assert ts.compare_states(sv, (got_re, got_im)) <= bar
    ore, oim = re.copy(), im.copy()
    ob.run_circuit(to_oracle(fused), ore, oim)
    assert np.abs((got_re - ore) + 1j * (got_im - oim)).max() <= bar
    info = plan.info()
    if info["swaps"]:
        assert rep["exchanged_bytes"] > 0


@pytest.mark.parametrize("kind,n,depth,kmax,prec,g", [("qft", 16, 1, 5, "f64", 2), ("rqc", 16, 6, 3, "f64", 1),
                                                      ("qaoa", 18, 3, 4, "f32", 2), ("hes", 16, 3, 5, "f32", 3)])
def test_vshard_forced_passes(kind, n, depth, kmax, prec, g, monkeypatch):
    """Every local run of a shard executes as a tile-pass program (forced)."""
    monkeypatch.setenv("TSG_PASS_FORCE", "1")
    c = ts.gen_benchmark(kind, n, depth, 7)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    re, im = random_state(n, 4)
    got_re, got_im, _ = ts.vshard_run(ts.ShardPlan(fused, g), re, im, prec)
    monkeypatch.delenv("TSG_PASS_FORCE")
    monkeypatch.setenv("TSG_NO_PASS", "1")
    sv = ts.Statevector(n, prec).upload(re, im)
    ts.run_circuit(fused, sv)
    assert ts.compare_states(sv, (got_re, got_im)) <= (1e-10 if prec == "f64" else 1e-5)


def test_qft_sharded_analytic():
    n, g, x = 18, 3, 0x2A5A5
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", n), ts.FusionConfig(k_max=5))
    re = np.zeros(1 << n)
    im = np.zeros(1 << n)
    re[x] = 1.0
    got_re, got_im, _ = ts.vshard_run(ts.ShardPlan(fused, g), re, im)
    y = np.arange(1 << n)
    want = np.exp(2j * np.pi * ((x * y) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
    assert np.abs(got_re + 1j * got_im - want).max() <= 1e-10


def test_dist_world_one():
    n = 14
    fused, _ = ts.run_fusion(ts.gen_benchmark("rqc", n, 6, 2), ts.FusionConfig(k_max=4))
    plan = ts.ShardPlan(fused, 0)
    uid = ts.DistState.unique_id()
    d = ts.DistState(n, 0, 0, uid)
    d.init_basis(5)
    rep = d.run(plan)
    assert rep["exchanged_bytes"] == 0
    re, im = d.download_local()
    sv = ts.Statevector(n, "f64").init_basis(5)
    ts.run_circuit(fused, sv)
    assert ts.compare_states(sv, (re, im)) <= 1e-12
    assert abs(d.local_sumsq() - 1.0) < 1e-9
