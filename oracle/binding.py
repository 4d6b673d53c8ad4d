"""ctypes binding of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle.so`` (the SPEC restatement, see oracle.cpp) and, when
present, ``oracle/_ref/libtsref.so`` (the reference's own gatecore/circuit
sources compiled unmodified).  Imported only by tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg.  Matrices cross the boundary as numpy
complex128 arrays (row-major, 2^k x 2^k); states as (re, im) numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtsref.so")

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p

MODES = {"none": 0, "size": 1, "size-only": 1, "adaptive": 2}


def build(ref: bool = False) -> None:
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _load():
    if not os.path.exists(LIB_PATH):
        build(ref=False)
    lib = C.CDLL(LIB_PATH)
    lib.orc_last_error.restype = C.c_char_p
    lib.orc_circuit_new.restype = _vp
    lib.orc_circuit_new.argtypes = [C.c_int]
    lib.orc_circuit_free.argtypes = [_vp]
    lib.orc_circuit_add_named.argtypes = [_vp, C.c_char_p, _dp, C.c_int, _ip, C.c_int]
    lib.orc_circuit_add_matrix.argtypes = [_vp, C.c_int, _ip, _dp]
    for f in ("orc_circuit_n_qubits", "orc_circuit_n_gates"):
        getattr(lib, f).argtypes = [_vp]
    lib.orc_circuit_gate_k.argtypes = [_vp, C.c_int]
    lib.orc_circuit_gate_targets.argtypes = [_vp, C.c_int, _ip]
    lib.orc_circuit_gate_matrix.argtypes = [_vp, C.c_int, _dp]
    lib.orc_circuit_gate_name.argtypes = [_vp, C.c_int]
    lib.orc_circuit_gate_name.restype = C.c_char_p
    lib.orc_gen_benchmark.argtypes = [C.c_char_p, C.c_int, C.c_int, _u64, C.POINTER(_vp)]
    lib.orc_random_unitary.argtypes = [C.c_int, _u64, C.c_int, _dp]
    lib.orc_prng_stream.argtypes = [_u64, C.c_int, C.POINTER(_u64), _dp]
    lib.orc_classify.argtypes = [C.c_double, C.c_double, C.c_double]
    lib.orc_profile.argtypes = [C.c_int, _dp, C.c_double, C.c_double, C.POINTER(C.c_uint8), C.POINTER(_u64)]
    lib.orc_is_unitary.argtypes = [C.c_int, _dp, C.c_double]
    lib.orc_fuse.argtypes = [C.c_int, _ip, _dp, C.c_int, _ip, _dp, _ip, _ip, _dp]
    lib.orc_expand.argtypes = [C.c_int, _ip, _dp, C.c_int, _ip, _dp]
    lib.orc_split.argtypes = [C.c_int, _ip, C.c_int, _ip]
    lib.orc_masks.argtypes = [C.c_int, _ip, C.c_int, C.c_int, C.POINTER(_u64), _ip]
    lib.orc_enumerate_indices.argtypes = [C.c_int, _ip, C.c_int, C.c_int, C.POINTER(_u64)]
    lib.orc_plan_entry_count.argtypes = [C.c_int, _dp, C.c_double, C.c_double, _ip]
    lib.orc_apply.argtypes = [C.c_int, C.c_int, _ip, _dp, C.c_int, C.c_double, C.c_double, _dp, _vp, _vp,
                              C.c_int, _u64, _u64]
    lib.orc_reference_apply.argtypes = [C.c_int, C.c_int, _ip, _dp, _vp, _vp, C.c_int]
    lib.orc_run_circuit.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                    C.c_int, _dp]
    lib.orc_run_circuit_slice.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, _u64,
                                          _u64, _dp]
    lib.orc_reference_run.argtypes = [_vp, _vp, _vp, C.c_int]
    lib.orc_norm.argtypes = [_vp, _vp, _u64, C.c_int]
    lib.orc_norm.restype = C.c_double
    lib.orc_compare.argtypes = [_dp, _dp, _dp, _dp, _u64]
    lib.orc_compare.restype = C.c_double
    lib.orc_run_fusion.argtypes = [_vp, _ip, C.c_int64, _dp, _vp, C.POINTER(_vp), C.POINTER(C.c_int64), _dp]
    lib.orc_cost_model_parse.argtypes = [C.c_char_p, C.POINTER(_vp)]
    lib.orc_cost_model_free.argtypes = [_vp]
    lib.orc_estimate_cost.argtypes = [_vp, C.c_int, _u64, C.c_int, C.c_int, _dp]
    return lib


LIB = _load()


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, LIB.orc_last_error().decode())


def _ints(xs):
    arr = (C.c_int * max(1, len(xs)))(*xs)
    return arr


def _mat_in(m: np.ndarray):
    a = np.ascontiguousarray(np.asarray(m, dtype=np.complex128)).view(np.float64)
    return a, a.ctypes.data_as(_dp)


def _mat_out(k: int):
    a = np.zeros((1 << k) * (1 << k) * 2, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _as_matrix(flat: np.ndarray, k: int) -> np.ndarray:
    return flat.view(np.complex128).reshape(1 << k, 1 << k).copy()


# ------------------------------------------------------------------ circuits
class Circuit:
    """Oracle-side circuit: list of (targets, matrix, name)."""

    def __init__(self, n: int = 0, handle=None):
        self.h = handle if handle is not None else LIB.orc_circuit_new(n)

    def __del__(self):
        if getattr(self, "h", None):
            LIB.orc_circuit_free(self.h)
            self.h = None

    def add(self, name: str, qubits, params=()):
        p = (C.c_double * max(1, len(params)))(*params)
        _check(LIB.orc_circuit_add_named(self.h, name.encode(), p, len(params), _ints(qubits), len(qubits)))
        return self

    def add_matrix(self, qubits, m):
        a, pm = _mat_in(m)
        _check(LIB.orc_circuit_add_matrix(self.h, len(qubits), _ints(qubits), pm))
        return self

    @property
    def n_qubits(self) -> int:
        return LIB.orc_circuit_n_qubits(self.h)

    def __len__(self) -> int:
        return LIB.orc_circuit_n_gates(self.h)

    def gate(self, i: int):
        k = LIB.orc_circuit_gate_k(self.h, i)
        t = (C.c_int * k)()
        LIB.orc_circuit_gate_targets(self.h, i, t)
        a, pm = _mat_out(k)
        LIB.orc_circuit_gate_matrix(self.h, i, pm)
        return list(t), _as_matrix(a, k), LIB.orc_circuit_gate_name(self.h, i).decode()

    def gates(self):
        return [self.gate(i) for i in range(len(self))]


def gen_benchmark(kind: str, n: int, depth: int = 1, seed: int = 0) -> Circuit:
    h = _vp()
    _check(LIB.orc_gen_benchmark(kind.encode(), n, depth, seed, C.byref(h)))
    return Circuit(handle=h.value)


# ------------------------------------------------------------------ gatecore
def random_unitary(k: int, seed: int, skip: int = 0) -> np.ndarray:
    a, pm = _mat_out(k)
    _check(LIB.orc_random_unitary(k, seed, skip, pm))
    return _as_matrix(a, k)


def prng_stream(seed: int, count: int):
    u = (_u64 * count)()
    nrm = np.zeros(count)
    LIB.orc_prng_stream(seed, count, u, nrm.ctypes.data_as(_dp))
    return list(u), nrm


def classify(x: float, zt: float = 1e-8, ot: float = 1e-8) -> int:
    return LIB.orc_classify(x, zt, ot)


def profile(m: np.ndarray, zt: float = 1e-8, ot: float = 1e-8):
    k = int(np.log2(m.shape[0]))
    a, pm = _mat_in(m)
    kinds = np.zeros(2 * m.size, dtype=np.uint8)
    cnt = (_u64 * 4)()
    _check(LIB.orc_profile(k, pm, zt, ot, kinds.ctypes.data_as(C.POINTER(C.c_uint8)), cnt))
    return kinds.reshape(m.size, 2), {"general": cnt[0], "one": cnt[1], "minus_one": cnt[2], "op_count": cnt[3]}


def is_unitary(m: np.ndarray, tol: float) -> bool:
    a, pm = _mat_in(m)
    return bool(LIB.orc_is_unitary(int(np.log2(m.shape[0])), pm, tol))


def fuse(t1, m1, t2, m2):
    a1, p1 = _mat_in(m1)
    a2, p2 = _mat_in(m2)
    u = sorted(set(t1) | set(t2))
    ok = C.c_int()
    ot = (C.c_int * max(1, len(u)))()
    if len(u) > 12:
        a, pm = _mat_out(1)
    else:
        a, pm = _mat_out(len(u))
    _check(LIB.orc_fuse(len(t1), _ints(t1), p1, len(t2), _ints(t2), p2, C.byref(ok), ot, pm))
    return list(ot)[: ok.value], _as_matrix(a, ok.value)


def expand(t, m, union):
    a, pm = _mat_in(m)
    o, po = _mat_out(len(union))
    _check(LIB.orc_expand(len(t), _ints(t), pm, len(union), _ints(union), po))
    return _as_matrix(o, len(union))


def split_qubits(targets, s: int):
    out = (C.c_int * (3 + len(targets)))()
    _check(LIB.orc_split(len(targets), _ints(targets), s, out))
    kl, kh = out[0], out[1]
    return {"k_L": kl, "k_H": kh, "lower_region": out[2], "lower": list(out[3:3 + kl]),
            "higher": list(out[3 + kl:3 + kl + kh])}


def build_masks(targets, s: int, n: int):
    out = (_u64 * 16)()
    cnt = C.c_int()
    _check(LIB.orc_masks(len(targets), _ints(targets), s, n, out, C.byref(cnt)))
    return list(out)[: cnt.value]


def enumerate_indices(targets, s: int, n: int) -> np.ndarray:
    out = np.zeros(1 << n, dtype=np.uint64)
    _check(LIB.orc_enumerate_indices(len(targets), _ints(targets), s, n, out.ctypes.data_as(C.POINTER(_u64))))
    return out


def plan_entry_count(m: np.ndarray, zt=1e-8, ot=1e-8) -> int:
    a, pm = _mat_in(m)
    out = C.c_int()
    _check(LIB.orc_plan_entry_count(int(np.log2(m.shape[0])), pm, zt, ot, C.byref(out)))
    return out.value


# --------------------------------------------------------------------- state
def _prec(re: np.ndarray) -> int:
    return 64 if re.dtype == np.float64 else 32


def apply_kernel(n, targets, m, re, im, s=0, zt=1e-8, ot=1e-8, override=None, t_begin=0, t_end=None):
    a, pm = _mat_in(m)
    po = None
    if override is not None:
        ao, po = _mat_in(override)
    if t_end is None:
        t_end = 1 << (n - len(targets) - s)
    _check(LIB.orc_apply(n, len(targets), _ints(targets), pm, s, zt, ot, po, re.ctypes.data, im.ctypes.data,
                         _prec(re), t_begin, t_end))


def reference_apply(n, targets, m, re, im):
    a, pm = _mat_in(m)
    _check(LIB.orc_reference_apply(n, len(targets), _ints(targets), pm, re.ctypes.data, im.ctypes.data, _prec(re)))


def run_circuit(c: Circuit, re, im, threads=1, s=0, zt=1e-8, ot=1e-8, g_begin=0, g_end=-1):
    times = np.zeros(2)
    _check(LIB.orc_run_circuit(c.h, re.ctypes.data, im.ctypes.data, _prec(re), threads, s, zt, ot, g_begin, g_end,
                               times.ctypes.data_as(_dp)))
    return {"planning_s": float(times[0]), "execution_s": float(times[1])}


def run_circuit_slice(c: Circuit, re, im, slice_: int, n_slices: int, threads=1, s=0, zt=1e-8, ot=1e-8):
    """Every gate of `c` over stratum `slice_` of `n_slices` equal parts of its
    group range (a bounded, stratified sample of run_circuit's work)."""
    times = np.zeros(2)
    _check(LIB.orc_run_circuit_slice(c.h, re.ctypes.data, im.ctypes.data, _prec(re), threads, s, zt, ot, slice_,
                                     n_slices, times.ctypes.data_as(_dp)))
    return {"planning_s": float(times[0]), "execution_s": float(times[1])}


def reference_run(c: Circuit, re, im):
    _check(LIB.orc_reference_run(c.h, re.ctypes.data, im.ctypes.data, _prec(re)))


def norm(re, im) -> float:
    return LIB.orc_norm(re.ctypes.data, im.ctypes.data, re.size, _prec(re))


def compare_states(ar, ai, br, bi) -> float:
    ar, ai, br, bi = (np.ascontiguousarray(x, dtype=np.float64) for x in (ar, ai, br, bi))
    return LIB.orc_compare(ar.ctypes.data_as(_dp), ai.ctypes.data_as(_dp), br.ctypes.data_as(_dp),
                           bi.ctypes.data_as(_dp), ar.size)


def zero_state(n: int, dtype=np.float64):
    re = np.zeros(1 << n, dtype=dtype)
    im = np.zeros(1 << n, dtype=dtype)
    re[0] = 1.0
    return re, im


# -------------------------------------------------------------------- fusion
class CostModel:
    def __init__(self, text: str):
        h = _vp()
        _check(LIB.orc_cost_model_parse(text.encode(), C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            LIB.orc_cost_model_free(self.h)
            self.h = None

    def estimate(self, k: int, ops: int, threads: int, n: int) -> float:
        out = C.c_double()
        _check(LIB.orc_estimate_cost(self.h, k, ops, threads, n, C.byref(out)))
        return out.value


def run_fusion(c: Circuit, mode="size", k_max=5, max_op_count=None, agglomerative=True, multi_traversal=True,
               zero_tol=1e-8, one_tol=1e-8, max_traversals=64, threads=1, cost_model: CostModel | None = None):
    ci = _ints([MODES[mode], k_max, int(agglomerative), int(multi_traversal), max_traversals, threads])
    cd = (C.c_double * 2)(zero_tol, one_tol)
    out = _vp()
    st = (C.c_int64 * 3)()
    sd = (C.c_double * 2)()
    _check(LIB.orc_run_fusion(c.h, ci, -1 if max_op_count is None else max_op_count, cd,
                              cost_model.h if cost_model else None, C.byref(out), st, sd))
    stats = {"original_gate_count": st[0], "fused_block_count": st[1], "total_op_count": st[2],
             "compression_ratio": sd[0], "fusion_wall_time": sd[1]}
    return Circuit(handle=out.value), stats


# ------------------------------------------------------- reference (_ref) ---
def load_ref():
    """The reference's own gatecore/circuit build, or None when absent."""
    if not os.path.exists(REF_PATH):
        return None
    lib = C.CDLL(REF_PATH)
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_named_gate.argtypes = [C.c_char_p, _dp, C.c_int, _ip, C.c_int, _ip, _ip, _dp]
    lib.ref_random_unitary.argtypes = [C.c_int, _u64, C.c_int, _dp]
    lib.ref_prng_stream.argtypes = [_u64, C.c_int, C.POINTER(_u64), _dp]
    lib.ref_classify.argtypes = [C.c_double, C.c_double, C.c_double]
    lib.ref_profile.argtypes = [C.c_int, _dp, C.c_double, C.c_double, C.POINTER(C.c_uint8), C.POINTER(_u64)]
    lib.ref_is_unitary.argtypes = [C.c_int, _dp, C.c_double]
    lib.ref_fuse.argtypes = [C.c_int, _ip, _dp, C.c_int, _ip, _dp, _ip, _ip, _dp]
    lib.ref_expand.argtypes = [C.c_int, _ip, _dp, C.c_int, _ip, _dp]
    lib.ref_make_gate_arg_order.argtypes = [C.c_int, _ip, _dp, _ip, _dp]
    lib.ref_parse_count.argtypes = [C.c_char_p, _ip]
    return lib
