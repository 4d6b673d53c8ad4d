"""k_stream_dmma tile copies through TMA tensor maps (dmma_tma_plan,
apply_impl.cuh) against the CPU oracle, in every TSG_DMMA_TMA mode:
0 per-chunk bulk copies, 1 tensor-map loads for the direct-out kernels (the
default), 3 tensor-map loads and write-backs for every kernel.

The geometries cover one unpadded run (targets 3..7), padded 256-byte chunks
(targets 0..4: box wider than the chunk, zero-filled padding that stores
skip), runs of consecutive high qubits (one copy per tile), scattered high
qubits (several copies per tile), controls in the run and in the tile base,
complex64 4- and 5-qubit products on the DMMA pipe (TSG_UMMA=0), and
4-qubit write-back kernels whose runs fit one box row (mode 3).  The
modes run in subprocesses: the mode is read once per process.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WORKER = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import random_gate_matrix, random_state
n = 16
cases = [
    ("f64", [3, 4, 5, 6, 7], "dense"), ("f64", [0, 1, 2, 3, 4], "dense"), ("f64", [11, 12, 13, 14, 15], "dense"),
    ("f64", [6, 9, 12, 14, 15], "dense"), ("f64", [1, 6, 9, 13, 15], "controlled"), ("f64", [0, 2, 7, 10, 13], "perm"),
    ("f64", [2, 5, 8, 12], "dense"), ("f64", [8, 10, 12, 14], "controlled"), ("f64", [4, 9, 13], "dense"),
    ("f32", [0, 1, 2, 3, 4], "dense"), ("f32", [5, 8, 11, 13, 15], "dense"), ("f32", [3, 7, 10, 14], "dense"),
    ("f64", [8, 9, 10, 11], "dense"), ("f64", [7, 9, 11, 13], "dense"),  # write-back kernels, 128-amplitude runs
]
out = []
for i, (prec, targets, kind) in enumerate(cases):
    m = random_gate_matrix(len(targets), 300 + i, kind)
    dt = np.float64 if prec == "f64" else np.float32
    re, im = random_state(n, 40 + i, dt)
    sv = ts.Statevector(n, prec).upload(re.astype(np.float64), im.astype(np.float64))
    plan = ts.KernelPlan(ts.Gate(targets, m), n)
    ts.apply_kernel(plan, sv)
    ore, oim = re.copy(), im.copy()
    ob.apply_kernel(n, targets, m, ore, oim)
    d = ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64)))
    out.append([prec, targets, kind, d])
print("RESULT " + json.dumps(out))
"""


def _run(mode):
    env = dict(os.environ, TSG_DMMA_TMA=str(mode), TSG_DMMA_DEBUG="1", TSG_UMMA="0")
    r = subprocess.run([sys.executable, "-c", _WORKER, ROOT], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1][7:])
    dbg = [ln for ln in r.stderr.splitlines() if ln.startswith("dmma ")]
    tma = [int(tok.split("=")[1]) for ln in dbg for tok in ln.split() if tok.startswith("tma=")]
    tpose = [int(tok.split("=")[1]) for ln in dbg for tok in ln.split() if tok.startswith("tpose=")]
    return res, tma, tpose


def test_dmma_tma_modes_match_oracle():
    counts = {}
    for mode in (0, 1, 3):
        res, tma, tpose = _run(mode)
        for prec, targets, kind, d in res:
            assert d <= (1e-12 if prec == "f64" else 1e-5), (mode, prec, targets, kind, d)
        assert len(tma) >= 8, tma  # (controlled and permutation cases may take other kernels)
        counts[mode] = sum(t > 0 for t in tma)
        if mode == 1:
            assert counts[1] >= 8, str(tma)  # the 5-qubit complex128 and 4-5 qubit complex64 products
            assert max(tma) > 1, tma  # scattered high targets: several tensor copies per tile
            # targets on qubit 0 (complex128 0..4, complex64 0..4): the transposed product
            assert sum(tpose) >= 2, tpose
    assert counts[0] == 0
    assert counts[3] >= counts[1] + 2, counts  # write-back (ks 3-4 complex128) kernels through the maps too
