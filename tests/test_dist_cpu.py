"""Host side of the multi-process (one process per GPU) path, on CPU:

* the shared-memory rendezvous the ranks of one box meet in (barrier +
  payload slots), world 2 and 4, its id broadcast over gloo exactly as
  bench.py / DistState users do;
* the shard planner's pipelining contract: an exchange marked pipelined
  leaves the slab bits T alone and the segment after it never touches T.
"""
import os
import socket

import numpy as np
import pytest

import paper_2503_19894_b200 as ts


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rv_worker(rank, world, port, iters, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        obj = [ts.DistState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        q.put((rank, ts.rendezvous_selftest(obj[0], rank, world, iters)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_rendezvous_barrier_and_slots(world):
    import torch.multiprocessing as mp

    iters = 300
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rv_worker, args=(r, world, port, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = world * 1000 * (iters * (iters - 1) // 2) + iters * (world * (world - 1) // 2)
    got = dict(q.get(timeout=10) for _ in range(world))
    assert all(v == want for v in got.values()), (got, want)


def test_rendezvous_rejects_bad_ids():
    with pytest.raises(ts.ConfigError):
        ts.rendezvous_selftest(b"no-leading-slash".ljust(128, b"\0"), 0, 1, 1)
    with pytest.raises(ts.ConfigError):
        ts.rendezvous_selftest(ts.DistState.unique_id(), 2, 2, 1)


@pytest.mark.parametrize("kind,n,depth,g", [("qft", 20, 1, 2), ("rqc", 20, 8, 3), ("qaoa", 20, 3, 2),
                                            ("hes", 20, 3, 3)])
def test_pipelined_exchanges_respect_slab_bits(kind, n, depth, g):
    fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 3), ts.FusionConfig(k_max=5))
    plan = ts.ShardPlan(fused, g, pipeline_bits=2)
    info = plan.info()
    nl = info["n_local"]
    tlo = nl - info["pipeline_bits"]
    ops = plan.ops()
    pipelined = 0
    for i, op in enumerate(ops):
        if op["kind"] != "swap" or op["pipeline_bits"] == 0:
            continue
        pipelined += 1
        assert all(lp < tlo for _, lp in op["swaps"])
        prefix = ops[i + 1:i + 1 + op["pipeline_ops"]]
        assert len(prefix) == op["pipeline_ops"] > 0
        for o in prefix:
            assert o["kind"] != "swap"
            assert all(t < tlo or t >= nl for t in o["gate"].targets), i
    assert pipelined == info["pipelined_exchanges"]
    assert info["exchanges"] >= info["pipelined_exchanges"]
    # no pipelining requested: every exchange is plain, the schedule otherwise identical
    flat = ts.ShardPlan(fused, g, pipeline_bits=0)
    assert flat.info()["pipelined_exchanges"] == 0 and flat.info()["pipeline_bits"] == 0


def test_pipeline_counts_on_the_c4_c5_configs():
    """The configurations the pipelining is for: RQC-33 / 8 ranks, TFIM-36 / 8."""
    out = {}
    for kind, n, depth in (("rqc", 33, 20), ("hes", 36, 20)):
        fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 42), ts.FusionConfig(k_max=5))
        info = ts.ShardPlan(fused, 3).info()
        out[kind] = (info["exchanges"], info["pipelined_exchanges"])
        assert info["exchanges"] > 0
    print(out)


def test_shard_aware_fusion_option():
    """FusionConfig.n_global: the fused gates never mix more of the top
    n_global qubits than their parts did; n_global = 0 is the reference's
    fusion bit for bit."""
    c = ts.gen_benchmark("qaoa", 16, 2, 3)
    base, _ = ts.run_fusion(c, ts.FusionConfig(k_max=5))
    same, _ = ts.run_fusion(c, ts.FusionConfig(k_max=5, n_global=0))
    assert [g.targets for g in base.gates()] == [g.targets for g in same.gates()]
    assert all(np.array_equal(a.matrix, b.matrix) for a, b in zip(base.gates(), same.gates()))
    aware, st = ts.run_fusion(c, ts.FusionConfig(k_max=5, n_global=2))
    assert st["fused_block_count"] >= len(base)
    assert max(len(g.targets) for g in aware.gates()) <= 5
