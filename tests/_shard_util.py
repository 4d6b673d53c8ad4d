"""Test harness: execute a product ShardPlan on CPU shards with the oracle.

Used two ways: all shards in one process (exchange = array swaps), and one
shard per gloo process (exchange = torch.distributed send/recv).  The oracle
applies each rank's gates (SPEC apply_kernel); the product supplies only the
schedule (tilesim/shard.hpp) -- the thing under test.
"""
import numpy as np

import paper_2503_19894_b200 as ts
from oracle import binding as ob


def half_indices(n_local: int, lp: int, v: int) -> np.ndarray:
    """Local indices whose bit lp equals v, in order of the remaining bits."""
    i = np.arange(1 << (n_local - 1), dtype=np.int64)
    low = i & ((1 << lp) - 1)
    return ((i >> lp) << (lp + 1)) | (v << lp) | low


def apply_gate(n_local, gate, re, im):
    if gate.k == 0:  # rank-wide phase
        d = complex(gate.matrix[0, 0])
        z = (re + 1j * im) * d
        re[:], im[:] = z.real, z.imag
        return
    ob.apply_kernel(n_local, gate.targets, gate.matrix, re, im)


def run_local_ops(plan: ts.ShardPlan, ops, i, rank, re, im, n_local):
    op = ops[i]
    if op["kind"] == "local":
        apply_gate(n_local, op["gate"], re, im)
    elif op["kind"] == "rank_block":
        apply_gate(n_local, plan.rank_subgate(i, rank), re, im)


def run_in_process(plan: ts.ShardPlan, re_full: np.ndarray, im_full: np.ndarray):
    """All 2^g shards in one process; returns the final state in logical order."""
    info = plan.info()
    nl, g = info["n_local"], info["n_global"]
    S, L = 1 << g, 1 << nl
    shards = [(re_full[s * L:(s + 1) * L].copy(), im_full[s * L:(s + 1) * L].copy()) for s in range(S)]
    ops = plan.ops()
    for i, op in enumerate(ops):
        if op["kind"] == "swap":
            for gp, lp in op["swaps"]:
                bit = gp - nl
                for s in range(S):
                    if (s >> bit) & 1:
                        continue
                    t = s | (1 << bit)
                    a1 = half_indices(nl, lp, 1)  # shard s (rank bit 0) sends its bit-lp = 1 half
                    a0 = half_indices(nl, lp, 0)
                    for arr in (0, 1):
                        tmp = shards[s][arr][a1].copy()
                        shards[s][arr][a1] = shards[t][arr][a0]
                        shards[t][arr][a0] = tmp
            continue
        for s in range(S):
            run_local_ops(plan, ops, i, s, shards[s][0], shards[s][1], nl)
    phys_re = np.concatenate([sh[0] for sh in shards])
    phys_im = np.concatenate([sh[1] for sh in shards])
    perm = ts.physical_permutation(plan.final_pos(), info["n"]).astype(np.int64)
    return phys_re[perm], phys_im[perm]


def run_rank(plan: ts.ShardPlan, rank: int, re: np.ndarray, im: np.ndarray, dist) -> None:
    """One shard per process; swaps over torch.distributed (gloo)."""
    import torch

    info = plan.info()
    nl = info["n_local"]
    ops = plan.ops()
    for i, op in enumerate(ops):
        if op["kind"] != "swap":
            run_local_ops(plan, ops, i, rank, re, im, nl)
            continue
        for gp, lp in op["swaps"]:
            bit = gp - nl
            peer = rank ^ (1 << bit)
            v = 1 - ((rank >> bit) & 1)  # the half this rank sends
            idx = half_indices(nl, lp, v)
            for arr in (re, im):
                send = torch.from_numpy(arr[idx].copy())
                recv = torch.empty_like(send)
                if rank < peer:
                    dist.send(send, peer)
                    dist.recv(recv, peer)
                else:
                    dist.recv(recv, peer)
                    dist.send(send, peer)
                arr[idx] = recv.numpy()
