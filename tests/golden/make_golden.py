"""Generate tests/golden/gatecore.json from the REFERENCE's own sources.

Runs only in the build container, where /root/reference exists: it builds
oracle/_ref/libtsref.so (proj/src/{complex_matrix,gate,circuit}.cpp compiled
unmodified, see oracle/Makefile) and records its outputs.  The fixtures pin
both the oracle restatement and the product's C++ gatecore bit-for-bit on
machines where the reference tree is absent (the GPU box).

Large matrices are stored as sha256 of their little-endian float64 bytes
(interleaved re, im; -0.0 normalised to +0.0, i.e. value equality).

    python tests/golden/make_golden.py
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import binding as ob  # noqa: E402


def mat_hash(m: np.ndarray) -> str:
    a = np.ascontiguousarray(np.asarray(m, dtype=np.complex128)).view(np.float64).copy()
    a[a == 0.0] = 0.0
    return hashlib.sha256(a.astype("<f8").tobytes()).hexdigest()


def mat_list(m: np.ndarray):
    return [[float(v.real), float(v.imag)] for v in np.asarray(m).reshape(-1)]


NAMED = [("x", [0], []), ("y", [0], []), ("z", [0], []), ("h", [0], []), ("s", [0], []), ("sdg", [0], []),
         ("t", [0], []), ("tdg", [0], []), ("rx", [0], [0.3]), ("ry", [0], [1.1]), ("rz", [0], [-0.7]),
         ("u3", [0], [0.3, 0.7, 1.1]), ("cx", [0, 1], []), ("cx", [1, 0], []), ("cx", [3, 1], []),
         ("cz", [0, 1], []), ("cp", [0, 1], [0.9]), ("cp", [2, 0], [1.7]), ("swap", [0, 1], []),
         ("ccx", [0, 1, 2], []), ("ccx", [2, 0, 1], []), ("ccx", [1, 3, 0], []), ("rx", [0], [1.5707963267948966]),
         ("ry", [0], [1.5707963267948966]), ("cp", [0, 1], [3.141592653589793 / 536870912])]

PARSE_CASES = [
    "qubits 1\nh 0\n",
    "qubits 2\ncx 0 1\n",
    "qubits 2\nh 5\n",
    "h 0\n",
    "qubits 2\nfoo 0\n",
    "qubits 2\nrx 0\n",
    "qubits 2\nrx(0.1,0.2) 0\n",
    "qubits 2\ncx 0 0\n",
    "qubits 2\nmatrix 1 0\n1,0 0,0\n0,0 1,0\n",
    "qubits 2\nmatrix 1 0\n1,0 1,0\n0,0 1,0\n",
    "qubits 3\nh 0 # comment\n\n  # blank\nccx 0 1 2\n",
    "qubits 63\n",
    "qubits 2\nqubits 2\n",
    "qubits 2\nh 0 1\n",
    "qubits 2\nrz(abc) 0\n",
]


def main():
    ob.build(ref=True)
    ref = ob.load_ref()
    assert ref is not None, "oracle/_ref/libtsref.so did not build"
    out = {"source": "reference proj/src/{complex_matrix,gate,circuit}.cpp via oracle/_ref", "named": [],
           "random_unitary": [], "prng": {}, "classify": [], "profile": [], "fuse": [], "expand": [],
           "parse": [], "arg_order": []}

    for name, q, p in NAMED:
        k = C.c_int()
        t = (C.c_int * 3)()
        m = np.zeros(2 * 64)
        pp = (C.c_double * 3)(*p)
        rc = ref.ref_named_gate(name.encode(), pp, len(p), ob._ints(q), len(q), C.byref(k), t, m.ctypes.data_as(ob._dp))
        assert rc == 0
        d = 1 << k.value
        mat = m[: 2 * d * d].view(np.complex128).reshape(d, d)
        out["named"].append({"name": name, "qubits": q, "params": p, "targets": list(t)[: k.value],
                             "matrix": mat_list(mat)})

    for k in range(1, 7):
        for seed, skip in ((42, 0), (7, 1)):
            m = np.zeros(2 * (1 << (2 * k)))
            ref.ref_random_unitary(k, seed, skip, m.ctypes.data_as(ob._dp))
            mat = m.view(np.complex128).reshape(1 << k, 1 << k)
            e = {"k": k, "seed": seed, "skip": skip, "sha256": mat_hash(mat)}
            if k <= 2:
                e["matrix"] = mat_list(mat)
            out["random_unitary"].append(e)

    u = (ob._u64 * 64)()
    nr = np.zeros(64)
    ref.ref_prng_stream(2024, 64, u, nr.ctypes.data_as(ob._dp))
    out["prng"] = {"seed": 2024, "u64": [str(x) for x in u], "normal": [float(x) for x in nr]}

    for x, zt, ot in [(0.0, 1e-8, 1e-8), (1.0, 1e-8, 1e-8), (0.7071067811865476, 1e-8, 1e-8), (-1.0, 1e-8, 1e-8),
                      (1.0, 0.0, 0.0), (5e-9, 1e-8, 1e-8), (1 - 5e-9, 1e-8, 1e-8), (-1 + 2e-8, 1e-8, 1e-8),
                      (0.5, 0.6, 0.6), (0.999, 0.0, 0.01)]:
        out["classify"].append({"x": x, "zt": zt, "ot": ot, "kind": ref.ref_classify(x, zt, ot)})

    for name, q, p in NAMED[:14]:
        g = [e for e in out["named"] if e["name"] == name and e["qubits"] == q][0]
        mat = np.array([complex(a, b) for a, b in g["matrix"]])
        d = int(round(np.sqrt(mat.size)))
        mat = mat.reshape(d, d)
        for zt, ot in ((1e-8, 1e-8), (1e-8, 0.0)):
            a, pm = ob._mat_in(mat)
            kinds = np.zeros(2 * mat.size, dtype=np.uint8)
            cnt = (ob._u64 * 4)()
            ref.ref_profile(int(np.log2(d)), pm, zt, ot, kinds.ctypes.data_as(C.POINTER(C.c_uint8)), cnt)
            out["profile"].append({"name": name, "qubits": q, "zt": zt, "ot": ot, "kinds": kinds.tolist(),
                                   "counts": [int(c) for c in cnt]})

    rng = np.random.default_rng(1234)
    for trial in range(40):
        k1 = int(rng.integers(1, 4))
        k2 = int(rng.integers(1, 4))
        t1 = sorted(rng.choice(7, k1, replace=False).tolist())
        t2 = sorted(rng.choice(7, k2, replace=False).tolist())
        s1, s2 = 500 + trial, 900 + trial
        m1 = np.zeros(2 * (1 << (2 * k1)))
        m2 = np.zeros(2 * (1 << (2 * k2)))
        ref.ref_random_unitary(k1, s1, 0, m1.ctypes.data_as(ob._dp))
        ref.ref_random_unitary(k2, s2, 0, m2.ctypes.data_as(ob._dp))
        u = sorted(set(t1) | set(t2))
        ok = C.c_int()
        ot = (C.c_int * 12)()
        om = np.zeros(2 * (1 << (2 * len(u))))
        rc = ref.ref_fuse(k1, ob._ints(t1), m1.ctypes.data_as(ob._dp), k2, ob._ints(t2), m2.ctypes.data_as(ob._dp),
                          C.byref(ok), ot, om.ctypes.data_as(ob._dp))
        assert rc == 0
        out["fuse"].append({"first": {"targets": t1, "seed": s1}, "second": {"targets": t2, "seed": s2},
                            "targets": list(ot)[: ok.value],
                            "sha256": mat_hash(om.view(np.complex128).reshape(1 << len(u), -1))})

    for (t, seed, uni) in [([1], 3, [0, 1]), ([0], 4, [0, 1]), ([0, 2], 5, [0, 1, 2]), ([1, 3], 6, [0, 1, 2, 3])]:
        k = len(t)
        m = np.zeros(2 * (1 << (2 * k)))
        ref.ref_random_unitary(k, seed, 0, m.ctypes.data_as(ob._dp))
        o = np.zeros(2 * (1 << (2 * len(uni))))
        ref.ref_expand(k, ob._ints(t), m.ctypes.data_as(ob._dp), len(uni), ob._ints(uni), o.ctypes.data_as(ob._dp))
        out["expand"].append({"targets": t, "seed": seed, "union": uni,
                              "sha256": mat_hash(o.view(np.complex128).reshape(1 << len(uni), -1))})

    for q, seed in [([1, 0], 11), ([2, 0, 1], 12), ([0, 2], 13), ([3, 1, 2], 14)]:
        k = len(q)
        m = np.zeros(2 * (1 << (2 * k)))
        ref.ref_random_unitary(k, seed, 0, m.ctypes.data_as(ob._dp))
        t = (C.c_int * k)()
        o = np.zeros_like(m)
        assert ref.ref_make_gate_arg_order(k, ob._ints(q), m.ctypes.data_as(ob._dp), t, o.ctypes.data_as(ob._dp)) == 0
        out["arg_order"].append({"qubits": q, "seed": seed, "targets": list(t),
                                 "sha256": mat_hash(o.view(np.complex128).reshape(1 << k, -1))})

    for text in PARSE_CASES:
        nq = C.c_int()
        cnt = ref.ref_parse_count(text.encode(), C.byref(nq))
        out["parse"].append({"text": text, "gates": cnt, "n_qubits": nq.value if cnt >= 0 else None,
                             "error": ref.ref_last_error().decode() if cnt < 0 else None})

    path = os.path.join(HERE, "gatecore.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
