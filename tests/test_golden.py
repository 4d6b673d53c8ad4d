"""Pin the oracle and the product's C++ gatecore to the REFERENCE's own outputs.

tests/golden/gatecore.json was produced by tests/golden/make_golden.py from the
reference sources compiled unmodified (oracle/_ref).  Every comparison is
bit-exact (value equality; -0.0 == +0.0).  When oracle/_ref is present (the
build container) the same checks also run live against it.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests.golden.make_golden import mat_hash

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "gatecore.json")))


def _mat(lst):
    a = np.array([complex(r, i) for r, i in lst])
    d = int(round(np.sqrt(a.size)))
    return a.reshape(d, d)


@pytest.mark.parametrize("case", GOLD["named"], ids=lambda c: f"{c['name']}{c['qubits']}")
def test_named_gates(case):
    want = _mat(case["matrix"])
    n = max(case["qubits"]) + 1
    o = ob.Circuit(n).add(case["name"], case["qubits"], case["params"])
    t, m, _ = o.gate(0)
    assert t == case["targets"] and np.array_equal(m, want)
    g = ts.make_named_gate(case["name"], case["params"], case["qubits"])
    assert g.targets == case["targets"] and np.array_equal(g.matrix, want)


@pytest.mark.parametrize("case", GOLD["random_unitary"], ids=lambda c: f"k{c['k']}s{c['seed']}")
def test_random_unitary(case):
    m = ob.random_unitary(case["k"], case["seed"], case["skip"])
    assert mat_hash(m) == case["sha256"]
    if "matrix" in case:
        assert np.array_equal(m, _mat(case["matrix"]))


def test_prng_stream():
    u, nrm = ob.prng_stream(GOLD["prng"]["seed"], 64)
    assert [str(x) for x in u] == GOLD["prng"]["u64"]
    assert np.array_equal(nrm, np.array(GOLD["prng"]["normal"]))


def test_classify():
    for c in GOLD["classify"]:
        assert ob.classify(c["x"], c["zt"], c["ot"]) == c["kind"], c


def test_profiles():
    named = {(e["name"], tuple(e["qubits"])): _mat(e["matrix"]) for e in GOLD["named"]}
    for c in GOLD["profile"]:
        m = named[(c["name"], tuple(c["qubits"]))]
        kinds, cnt = ob.profile(m, c["zt"], c["ot"])
        assert kinds.reshape(-1).tolist() == c["kinds"]
        assert [cnt["general"], cnt["one"], cnt["minus_one"], cnt["op_count"]] == c["counts"]


@pytest.mark.parametrize("case", GOLD["fuse"], ids=lambda c: f"{c['first']['targets']}x{c['second']['targets']}")
def test_fuse_matrices(case):
    a, b = case["first"], case["second"]
    m1 = ob.random_unitary(len(a["targets"]), a["seed"])
    m2 = ob.random_unitary(len(b["targets"]), b["seed"])
    u, f = ob.fuse(a["targets"], m1, b["targets"], m2)
    assert u == case["targets"] and mat_hash(f) == case["sha256"]
    # product: a 2-gate circuit fused into one block is exactly fuse_matrices(first, second)
    n = max(u) + 1
    c = ts.Circuit(n).add_matrix(a["targets"], m1).add_matrix(b["targets"], m2)
    fused, _ = ts.run_fusion(c, ts.FusionConfig(k_max=len(u), agglomerative=False))
    if len(fused) == 1:
        g = fused.gate(0)
        assert g.targets == case["targets"] and mat_hash(g.matrix) == case["sha256"]


def test_expand():
    for c in GOLD["expand"]:
        m = ob.random_unitary(len(c["targets"]), c["seed"])
        assert mat_hash(ob.expand(c["targets"], m, c["union"])) == c["sha256"]


def test_arg_order():
    for c in GOLD["arg_order"]:
        m = ob.random_unitary(len(c["qubits"]), c["seed"])
        n = max(c["qubits"]) + 1
        o = ob.Circuit(n).add_matrix(c["qubits"], m)
        t, mm, _ = o.gate(0)
        assert t == c["targets"] and mat_hash(mm) == c["sha256"]
        g = ts.Circuit(n).add_matrix(c["qubits"], m).gate(0)
        assert g.targets == c["targets"] and mat_hash(g.matrix) == c["sha256"]


@pytest.mark.parametrize("case", GOLD["parse"], ids=lambda c: repr(c["text"][:18]))
def test_parse_matches_reference(case):
    if case["gates"] < 0:
        with pytest.raises(ts.ParseError) as e:
            ts.parse_circuit(case["text"])
        assert str(e.value) == case["error"]
    else:
        c = ts.parse_circuit(case["text"])
        assert len(c) == case["gates"] and c.n_qubits == case["n_qubits"]


REF = ob.load_ref()


@pytest.mark.skipif(REF is None, reason="oracle/_ref not built (no /root/reference here)")
def test_live_reference_random_fuse():
    """Live: 300 random fusions, restatement vs the reference build, bit-exact."""
    rng = np.random.default_rng(99)
    for trial in range(300):
        k1, k2 = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        t1 = sorted(rng.choice(8, k1, replace=False).tolist())
        t2 = sorted(rng.choice(8, k2, replace=False).tolist())
        if len(set(t1) | set(t2)) > 6:
            continue
        m1, m2 = ob.random_unitary(k1, trial), ob.random_unitary(k2, trial + 5000)
        u, f = ob.fuse(t1, m1, t2, m2)
        ok = C.c_int()
        ot = (C.c_int * 12)()
        om = np.zeros(2 * (1 << (2 * len(u))))
        a1, p1 = ob._mat_in(m1)
        a2, p2 = ob._mat_in(m2)
        assert REF.ref_fuse(k1, ob._ints(t1), p1, k2, ob._ints(t2), p2, C.byref(ok), ot, om.ctypes.data_as(ob._dp)) == 0
        assert np.array_equal(om.view(np.complex128).reshape(f.shape), f)
