"""The multi-process data plane on the device.

* Virtual shards (one process): tsg_vshard_run drives the distributed
  exchange kernel itself (k_exchange, every virtual rank its share of the
  pairs, slab by slab) -- pipelined plans against the unsharded run.
* Real ranks: 2 and 4 processes, each with its own CUDA context and shard,
  peer shards mapped over CUDA IPC, exchanges in place over peer memory,
  ordered by interprocess events and the shared-memory rendezvous.  Only one
  B200 is available per run, so the ranks share it (the IPC, event and
  rendezvous paths are the same as across NVLink peers).  Shard invariance:
  the gathered state equals the one-GPU Program run within the north-star
  bars.
"""
import os
import socket

import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from tests._util import random_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,depth,prec,g", [("rqc", 18, 8, "f64", 2), ("qft", 18, 1, "f64", 3),
                                                 ("qaoa", 18, 3, "f32", 2), ("hes", 17, 4, "f64", 1)])
def test_vshard_pipelined_exchanges(kind, n, depth, prec, g):
    fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 9), ts.FusionConfig(k_max=5))
    plan = ts.ShardPlan(fused, g, pipeline_bits=2)
    re, im = random_state(n, 5)
    got_re, got_im, rep = ts.vshard_run(plan, re, im, prec)
    sv = ts.Statevector(n, prec).upload(re, im)
    ts.run_circuit(fused, sv)
    assert ts.compare_states(sv, (got_re, got_im)) <= (1e-10 if prec == "f64" else 1e-5)
    if plan.info()["exchanges"]:
        assert rep["exchanged_bytes"] > 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, kind, n, depth, prec, pipeline_bits, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 11), ts.FusionConfig(k_max=5))
        plan = ts.ShardPlan(fused, g, pipeline_bits=pipeline_bits)
        obj = [ts.DistState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        d = ts.DistState(n, g, rank, obj[0], prec, ts.Context(0))
        re, im = random_state(n, 21)
        L = 1 << (n - g)
        d.upload_local(re[rank * L:(rank + 1) * L], im[rank * L:(rank + 1) * L])
        rep = d.run(plan)
        rep2 = d.run(ts.ShardPlan(fused, g, pipeline_bits=pipeline_bits))  # a second plan: fresh schedule
        lre, lim = d.download_local()
        parts_re = [torch.empty(L, dtype=torch.float64) for _ in range(world)]
        parts_im = [torch.empty(L, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts_re, torch.from_numpy(lre))
        dist.all_gather(parts_im, torch.from_numpy(lim))
        d.close()
        if rank == 0:
            # the state after the circuit applied twice, in logical order:
            # physical index of logical x after two runs = pos2(pos1 map)...
            phys_re = np.concatenate([p.numpy() for p in parts_re])
            phys_im = np.concatenate([p.numpy() for p in parts_im])
            sv = ts.Statevector(n, prec).upload(re, im)
            prog = ts.Program(fused, prec)
            prog.run(sv)
            # the second run started from the first run's physical layout: its
            # logical qubit q sat at physical final_pos[q]; the plan treats the
            # input as logical order, so compare against the permuted circuit
            want_re, want_im = sv.download()
            pos = plan.final_pos()
            perm1 = ts.physical_permutation(pos, n).astype(np.int64)
            # after run 1: logical x at perm1[x].  Run 2 relabels again.
            st = ts.Statevector(n, prec).upload(want_re[np.argsort(perm1)], want_im[np.argsort(perm1)])
            prog.run(st)
            w2re, w2im = st.download()
            perm2 = perm1
            got = (phys_re + 1j * phys_im)[perm2]
            q.put({"diff": float(np.abs(got - (w2re + 1j * w2im)).max()), "exchanged": rep["exchanged_bytes"],
                   "exchange_s": rep["exchange_s"], "launches": rep["launches"], "second": rep2["launches"]})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind,n,depth,prec,pipeline_bits", [("rqc", 18, 8, "f64", 2), ("qft", 18, 1, "f64", 0),
                                                             ("qaoa", 18, 3, "f32", 2)])
def test_multiprocess_ranks_on_one_gpu(world, kind, n, depth, prec, pipeline_bits):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, kind, n, depth, prec, pipeline_bits, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for p in procs:
        if p.exitcode is None:
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = q.get(timeout=10)
    print(res)
    assert res["diff"] <= (1e-10 if prec == "f64" else 1e-5), res
    assert res["exchanged"] > 0 and res["exchange_s"] > 0


def _read_qsv1(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"QSV1"
    bits, n = raw[4], raw[5]
    dt = np.float64 if bits == 64 else np.float32
    a = np.frombuffer(raw[16:], dtype=dt)
    return a[: 1 << n].astype(np.float64), a[1 << n:].astype(np.float64)


def _dump_main(rank, world, port, path, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, g = 16, world.bit_length() - 1
        fused, _ = ts.run_fusion(ts.gen_benchmark("rqc", n, 6, 4), ts.FusionConfig(k_max=4))
        plan = ts.ShardPlan(fused, g)
        ctx = ts.Context(0)
        for i in range(2):
            obj = [ts.DistState.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            d = ts.DistState(n, g, rank, obj[0], "f64", ctx)
            if i == 0:
                d.init_basis(0x1234)
                d.run(plan)
                before = d.download_local()
                d.dump(path, plan.final_pos())
            else:
                pos = d.load(path)
                after = d.download_local()
            d.close()
            dist.barrier()
        ok = pos == plan.final_pos() and all(np.array_equal(a, b) for a, b in zip(before, after))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_sharded_qsv1_dump_load(tmp_path):
    """Sharded QSV1: every rank dumps its shard, fresh ranks load
    them back bit for bit; the host reassembles the logical state from the
    shard files and the layout's qubit map and matches the one-GPU run."""
    import torch.multiprocessing as mp

    world, n = 2, 16
    path = str(tmp_path / "state")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dump_main, args=(r, world, port, path, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = dict(q.get(timeout=10) for _ in range(world))
    assert all(res.values()), res
    layout = open(path + ".layout").read().split()
    pos = [int(x) for x in layout[layout.index("pos") + 1:]]
    shards = [_read_qsv1(f"{path}.r{r}") for r in range(world)]
    phys_re = np.concatenate([s[0] for s in shards])
    phys_im = np.concatenate([s[1] for s in shards])
    perm = ts.physical_permutation(pos, n).astype(np.int64)
    fused, _ = ts.run_fusion(ts.gen_benchmark("rqc", n, 6, 4), ts.FusionConfig(k_max=4))
    sv = ts.Statevector(n, "f64").init_basis(0x1234)
    ts.run_circuit(fused, sv)
    assert ts.compare_states(sv, (phys_re[perm], phys_im[perm])) <= 1e-12
