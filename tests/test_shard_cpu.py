"""Global-qubit sharding on CPU: the product's shard planner (tilesim/shard.hpp)
executed with the oracle's apply_kernel, in one process and over real gloo
processes (world size 2 and 4), against the unsharded oracle.

SURVEY.md §4: "a CPU sharded oracle that holds 2^g shard arrays ... must
match the unsharded result"; §8(e) exchange-free cases.
"""
import os
import socket

import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._shard_util import run_in_process, run_rank
from tests._util import random_state, to_oracle

CASES = [("qft", 10, 1, 4), ("rqc", 9, 6, 3), ("qaoa", 10, 2, 4), ("hes", 9, 3, 3), ("qvc", 8, 3, 2),
         ("iqp", 9, 3, 3), ("ala", 8, 3, 4)]


def _reference(c, fused, re, im):
    ore, oim = re.copy(), im.copy()
    ob.run_circuit(to_oracle(fused), ore, oim)
    return ore, oim


@pytest.mark.parametrize("kind,n,depth,kmax", CASES)
@pytest.mark.parametrize("g", [1, 2, 3])
def test_sharded_schedule_matches_unsharded(kind, n, depth, kmax, g):
    c = ts.gen_benchmark(kind, n, depth, 5)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
    if n - g < kmax:
        pytest.skip("gate wider than a shard")
    plan = ts.ShardPlan(fused, g)
    re, im = random_state(n, 11)
    want_re, want_im = _reference(c, fused, re, im)
    got_re, got_im = run_in_process(plan, re, im)
    assert np.abs((got_re - want_re) + 1j * (got_im - want_im)).max() <= 1e-12


def test_exchange_free_gates():
    """Diagonal / controlled gates on global qubits run as rank blocks: no swaps."""
    n = 8
    c = ts.Circuit(n)
    for q in range(n - 1):
        c.add("cp", [q, n - 1], [0.3 + q])  # every CP touches the top (global) qubit
    c.add("cz", [6, 7]).add("rz", [7], [0.4]).add("t", [6])
    c.add("cx", [7, 2])  # control on a global qubit: block-diagonal on it
    plan = ts.ShardPlan(c, 2)
    info = plan.info()
    assert info["swaps"] == 0 and info["rank_blocks"] >= n
    re, im = random_state(n, 2)
    want = _reference(c, c, re, im)
    got = run_in_process(plan, re, im)
    assert np.abs((got[0] - want[0]) + 1j * (got[1] - want[1])).max() <= 1e-12


def test_swap_eviction_is_belady_then_highest():
    n = 10
    # qubit 7 is used again soon: 6 is evicted first; qubit 9 (now at local 6)
    # is never used again, so it is the next victim (furthest next use)
    c = ts.Circuit(n).add("h", [9]).add("h", [8]).add("x", [7]).add("x", [0])
    plan = ts.ShardPlan(c, 2)
    swaps = [op["swaps"] for op in plan.ops() if op["kind"] == "swap"]
    assert swaps == [[(9, 6)], [(8, 6)]]
    assert plan.final_pos()[8] == 6 and plan.final_pos()[9] == 8 and plan.final_pos()[6] == 9
    # nothing used again: ties break to the highest free local position
    c2 = ts.Circuit(n).add("h", [9]).add("h", [8])
    assert [op["swaps"] for op in ts.ShardPlan(c2, 2).ops() if op["kind"] == "swap"] == [[(9, 7)], [(8, 7)]]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, n, depth, kmax, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        c = ts.gen_benchmark(kind, n, depth, 5)
        fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=kmax))
        plan = ts.ShardPlan(fused, g)
        re, im = random_state(n, 11)
        L = 1 << (n - g)
        lre, lim = re[rank * L:(rank + 1) * L].copy(), im[rank * L:(rank + 1) * L].copy()
        run_rank(plan, rank, lre, lim, dist)
        import torch

        parts_re = [torch.empty(L, dtype=torch.float64) for _ in range(world)]
        parts_im = [torch.empty(L, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts_re, torch.from_numpy(lre))
        dist.all_gather(parts_im, torch.from_numpy(lim))
        if rank == 0:
            phys_re = np.concatenate([p.numpy() for p in parts_re])
            phys_im = np.concatenate([p.numpy() for p in parts_im])
            perm = ts.physical_permutation(plan.final_pos(), n).astype(np.int64)
            want_re, want_im = _reference(c, fused, re, im)
            q.put(float(np.abs((phys_re[perm] - want_re) + 1j * (phys_im[perm] - want_im)).max()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind,n,depth,kmax", [("qft", 10, 1, 4), ("rqc", 10, 6, 3)])
def test_gloo_multiprocess(world, kind, n, depth, kmax):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, depth, kmax, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=10) <= 1e-12
