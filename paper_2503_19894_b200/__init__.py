"""tilesim-b200: the B200 (sm_100a) gate-application path of CAST/tilesim.

Python mirror of the reference's operator surface, bound through the C ABI of
``libtilesim_b200.so`` (include/tilesim_cuda.h).  Names follow the reference:

  gatecore / circuit  make_named_gate, gen_benchmark, parse_circuit,
                      serialize_circuit, Circuit               (proj/src/circuit.cpp,
                                                                SPEC.md:136-198)
  fusion              run_fusion, FusionConfig, CostModel, estimate_cost
                                                               
  kernel              plan_kernel -> KernelPlan, apply_kernel
  sim                 Statevector, init_zero_state, run_circuit, norm,
                      compare_states

There is no CPU fallback: device calls raise SimError on a host without a
CUDA device, and importing this package raises ImportError when the shared
library has not been built (``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtilesim_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` (no CPU fallback exists)")

_lib = C.CDLL(LIB_PATH)

_u64 = C.c_uint64
_i64 = C.c_int64
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class TilesimError(RuntimeError):
    code = 3


class ParseError(TilesimError):
    code = 1


class ConfigError(TilesimError):
    code = 2


class SimError(TilesimError):
    code = 3


_ERRORS = {1: ParseError, 2: ConfigError, 3: SimError}


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, TilesimError)(_lib.tsg_last_error().decode())


class PlanInfo(C.Structure):
    _fields_ = [("k", C.c_int), ("kernel_class", C.c_int), ("sub_k", C.c_int), ("n_controls", C.c_int),
                ("sparse", C.c_int), ("op_count", _u64), ("entry_ops", _u64), ("loop_count", _u64),
                ("touched_fraction", C.c_double), ("batched", C.c_int), ("controls", C.c_int * 12),
                ("sub_targets", C.c_int * 12)]


def _plan_info_dict(pi) -> dict:
    d = {f: getattr(pi, f) for f, _ in PlanInfo._fields_}
    d["kernel"] = KERNEL_CLASSES[pi.kernel_class]
    d["controls"] = list(pi.controls[:pi.n_controls])
    d["sub_targets"] = list(pi.sub_targets[:pi.sub_k])
    return d


class RunReport(C.Structure):
    _fields_ = [("planning_s", C.c_double), ("execution_s", C.c_double), ("gates", _u64), ("launches", _u64),
                ("bytes", _u64), ("touched_bytes", _u64), ("total_op_count", _u64), ("exchanged_bytes", _u64),
                ("exchange_s", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class StepInfo(C.Structure):
    _fields_ = [("kind", C.c_int), ("first_gate", _u64), ("n_gates", _u64), ("n_high", C.c_int),
                ("high", C.c_int * 16), ("kernel", C.c_char * 48)]


STEP_KINDS = ("gate", "diag_batch", "pass", "permute")


class _FusionConfigC(C.Structure):
    _fields_ = [("mode", C.c_int), ("k_max", C.c_int), ("max_op_count", _i64), ("agglomerative", C.c_int),
                ("multi_traversal", C.c_int), ("zero_tol", C.c_double), ("one_tol", C.c_double),
                ("max_traversals", C.c_int), ("threads", C.c_int), ("n_global", C.c_int)]


class _FusionStatsC(C.Structure):
    _fields_ = [("original_gate_count", _u64), ("fused_block_count", _u64), ("total_op_count", _u64),
                ("compression_ratio", C.c_double), ("fusion_wall_time", C.c_double)]


def _sig(name, args, res=C.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res


_sig("tsg_last_error", [], C.c_char_p)
_sig("tsg_version", [], C.c_char_p)
_sig("tsg_device_count", [_ip])
_sig("tsg_ctx_create", [C.c_int, C.POINTER(_vp)])
_sig("tsg_ctx_destroy", [_vp])
_sig("tsg_state_create", [_vp, C.c_int, C.c_int, C.POINTER(_vp)])
_sig("tsg_state_destroy", [_vp])
_sig("tsg_state_info", [_vp, _ip, _ip])
_sig("tsg_state_init_zero", [_vp])
_sig("tsg_state_init_basis", [_vp, _u64])
_sig("tsg_state_init_random", [_vp, _u64])
_sig("tsg_state_upload", [_vp, _dp, _dp])
_sig("tsg_state_upload_range", [_vp, _u64, _u64, _dp, _dp])
_sig("tsg_state_download", [_vp, _dp, _dp])
_sig("tsg_state_download_range", [_vp, _u64, _u64, _dp, _dp])
_sig("tsg_state_gather", [_vp, C.POINTER(_u64), _u64, _dp, _dp])
_sig("tsg_state_copy", [_vp, _vp])
_sig("tsg_state_dump", [_vp, C.c_char_p])
_sig("tsg_state_load", [_vp, C.c_char_p])
_sig("tsg_synchronize", [_vp])
_sig("tsg_timer_begin", [_vp])
_sig("tsg_timer_end", [_vp, _dp])
_sig("tsg_plan_create", [_vp, C.c_int, C.c_int, _ip, _dp, C.c_double, C.c_double, C.c_int, C.POINTER(_vp)])
_sig("tsg_plan_destroy", [_vp])
_sig("tsg_plan_info_get", [_vp, C.POINTER(PlanInfo)])
_sig("tsg_apply", [_vp, _vp, _dp, _u64, _u64])
_sig("tsg_norm", [_vp, _dp])
_sig("tsg_compare", [_vp, _dp, _dp, _dp])
_sig("tsg_compare_states", [_vp, _vp, _dp])
_sig("tsg_overlap", [_vp, _vp, _dp, _dp])
_sig("tsg_program_create", [_vp, _vp, C.c_double, C.c_double, C.c_int, C.POINTER(_vp)])
_sig("tsg_program_destroy", [_vp])
_sig("tsg_program_run", [_vp, _vp, C.c_int, C.POINTER(RunReport)])
_sig("tsg_program_enqueue", [_vp, _vp, C.c_int])
_sig("tsg_program_run_profiled", [_vp, _vp, _dp, C.POINTER(RunReport)])
_sig("tsg_program_gate_info", [_vp, _u64, C.POINTER(PlanInfo)])
_sig("tsg_program_step_count", [_vp, C.POINTER(_u64)])
_sig("tsg_program_step_info", [_vp, _u64, C.POINTER(StepInfo)])
_sig("tsg_program_pass_layouts", [_vp, _u64, C.POINTER(C.c_int), C.POINTER(C.c_int)])
_sig("tsg_program_jit_kernels", [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)])
_sig("tsc_plan_passes", [_vp, C.c_int, C.c_double, C.c_double, _ip, _ip, _ip, C.POINTER(_u64)])
_sig("tsg_ctx_info", [_vp, _ip, _ip])
_sig("tsg_bench_cost_model", [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _u64, C.POINTER(_vp)])
_sig("tsg_bench_cost_model_sms", [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _u64, _ip, C.c_int, C.POINTER(_vp)])
_sig("tsc_circuit_create", [C.c_int, C.POINTER(_vp)])
_sig("tsc_circuit_destroy", [_vp])
_sig("tsc_circuit_copy", [_vp, C.POINTER(_vp)])
_sig("tsc_circuit_add_named", [_vp, C.c_char_p, _dp, C.c_int, _ip, C.c_int])
_sig("tsc_circuit_add_matrix", [_vp, C.c_int, _ip, _dp])
_sig("tsc_circuit_n_qubits", [_vp, _ip])
_sig("tsc_circuit_n_gates", [_vp, C.POINTER(_u64)])
_sig("tsc_circuit_gate", [_vp, _u64, _ip, _ip, _dp])
_sig("tsc_circuit_gate_name", [_vp, _u64], C.c_char_p)
_sig("tsc_gen_benchmark", [C.c_char_p, C.c_int, C.c_int, _u64, C.POINTER(_vp)])
_sig("tsc_parse_circuit", [C.c_char_p, C.POINTER(_vp)])
_sig("tsc_serialize_circuit", [_vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)])
_sig("tsc_run_fusion", [_vp, C.POINTER(_FusionConfigC), _vp, C.POINTER(_vp), C.POINTER(_FusionStatsC)])
_sig("tsc_cost_model_parse", [C.c_char_p, C.POINTER(_vp)])
_sig("tsc_cost_model_destroy", [_vp])
_sig("tsc_cost_model_serialize", [_vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)])
_sig("tsc_estimate_cost", [_vp, C.c_int, _u64, C.c_int, C.c_int, _dp])

KERNEL_CLASSES = ("identity", "diagonal", "direct", "tile")


def version() -> str:
    return _lib.tsg_version().decode()


def device_count() -> int:
    n = C.c_int()
    _lib.tsg_device_count(C.byref(n))
    return n.value


def _ints(xs):
    xs = list(xs)
    return (C.c_int * max(1, len(xs)))(*xs)


def _matrix_arg(m) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(m, dtype=np.complex128))
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] & (a.shape[0] - 1):
        raise ConfigError("matrix must be square with a power-of-two dimension")
    return a.view(np.float64).reshape(-1)


def _read_text(fn, handle) -> str:
    need = C.c_size_t()
    _check(fn(handle, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(fn(handle, buf, need.value, C.byref(need)))
    return buf.value.decode()


# ============================================================ circuit IR ===
@dataclass
class Gate:
    """A k-qubit operator on strictly increasing targets (gate.hpp:17-24)."""
    targets: list
    matrix: np.ndarray
    name: str = ""

    @property
    def k(self) -> int:
        return len(self.targets)


class Circuit:
    """Program-ordered gate list (circuit.hpp:12-15), owned by the C++ side."""

    def __init__(self, n_qubits: int = 0, _handle=None):
        if _handle is None:
            h = _vp()
            _check(_lib.tsc_circuit_create(n_qubits, C.byref(h)))
            _handle = h.value
        self._h = _handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsc_circuit_destroy(self._h)
            self._h = None

    @property
    def n_qubits(self) -> int:
        n = C.c_int()
        _check(_lib.tsc_circuit_n_qubits(self._h, C.byref(n)))
        return n.value

    def __len__(self) -> int:
        n = _u64()
        _check(_lib.tsc_circuit_n_gates(self._h, C.byref(n)))
        return n.value

    def add(self, name: str, qubits, params=()):
        """make_named_gate(name, params, qubits) appended; qubits in argument order."""
        p = (C.c_double * max(1, len(params)))(*params)
        _check(_lib.tsc_circuit_add_named(self._h, name.encode(), p, len(params), _ints(qubits), len(qubits)))
        return self

    def add_matrix(self, qubits, matrix):
        """Raw unitary in the argument order of `qubits` (make_gate_arg_order)."""
        m = _matrix_arg(matrix)
        _check(_lib.tsc_circuit_add_matrix(self._h, len(qubits), _ints(qubits), m.ctypes.data_as(_dp)))
        return self

    def gate(self, i: int) -> Gate:
        k = C.c_int()
        _check(_lib.tsc_circuit_gate(self._h, i, C.byref(k), None, None))
        t = (C.c_int * k.value)()
        m = np.zeros(2 * (1 << (2 * k.value)))
        _check(_lib.tsc_circuit_gate(self._h, i, None, t, m.ctypes.data_as(_dp)))
        d = 1 << k.value
        return Gate(list(t), m.view(np.complex128).reshape(d, d).copy(),
                    _lib.tsc_circuit_gate_name(self._h, i).decode())

    def gates(self):
        return [self.gate(i) for i in range(len(self))]

    def copy(self) -> "Circuit":
        h = _vp()
        _check(_lib.tsc_circuit_copy(self._h, C.byref(h)))
        return Circuit(_handle=h.value)

    def serialize(self) -> str:
        return _read_text(_lib.tsc_serialize_circuit, self._h)


def gen_benchmark(kind: str, n: int, depth: int = 1, seed: int = 0) -> Circuit:
    """QFT ALA RQC QVC IQP HES and QAOA; recipes in DESIGN.md §3."""
    h = _vp()
    _check(_lib.tsc_gen_benchmark(kind.lower().encode(), n, depth, seed, C.byref(h)))
    return Circuit(_handle=h.value)


def parse_circuit(text: str) -> Circuit:
    h = _vp()
    _check(_lib.tsc_parse_circuit(text.encode(), C.byref(h)))
    return Circuit(_handle=h.value)


def serialize_circuit(c: Circuit) -> str:
    return c.serialize()


def make_named_gate(name: str, params, qubits) -> Gate:
    c = Circuit(max(qubits) + 1)
    c.add(name, qubits, params)
    return c.gate(0)


# ================================================================ fusion ===
@dataclass
class FusionConfig:
    """SPEC.md:311-315.  mode: 'none' | 'size-only' | 'adaptive'."""
    k_max: int = 5
    max_op_count: int | None = None
    mode: str = "size-only"
    agglomerative: bool = True
    multi_traversal: bool = True
    zero_tol: float = 1e-8
    one_tol: float = 1e-8
    max_traversals: int = 64
    threads: int = 1
    n_global: int = 0  # shard-aware fusion over the top n_global qubits (0: the reference's fusion)

    @staticmethod
    def paper_cpu() -> "FusionConfig":
        return FusionConfig(k_max=7, max_op_count=4096, mode="adaptive")

    def _c(self) -> _FusionConfigC:
        modes = {"none": 0, "size-only": 1, "size": 1, "adaptive": 2}
        if self.mode not in modes:
            raise ConfigError(f"unknown fusion mode {self.mode!r}")
        return _FusionConfigC(modes[self.mode], self.k_max, -1 if self.max_op_count is None else self.max_op_count,
                              int(self.agglomerative), int(self.multi_traversal), self.zero_tol, self.one_tol,
                              self.max_traversals, self.threads, self.n_global)


class CostModel:
    """Measured (k, op_count, threads) -> seconds-per-group table."""

    def __init__(self, text: str | None = None, _handle=None):
        if _handle is None:
            h = _vp()
            _check(_lib.tsc_cost_model_parse((text or "").encode(), C.byref(h)))
            _handle = h.value
        self._h = _handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsc_cost_model_destroy(self._h)
            self._h = None

    @staticmethod
    def load(path: str) -> "CostModel":
        if not os.path.exists(path):
            raise ParseError(f"cost model file not found: {path}")
        with open(path) as f:
            return CostModel(f.read())

    def save(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.serialize())

    def serialize(self) -> str:
        return _read_text(_lib.tsc_cost_model_serialize, self._h)

    def estimate(self, k: int, op_count: int, threads: int, n: int) -> float:
        out = C.c_double()
        _check(_lib.tsc_estimate_cost(self._h, k, op_count, threads, n, C.byref(out)))
        return out.value


def run_fusion(c: Circuit, cfg: FusionConfig | None = None, cost_model: CostModel | None = None):
    """run_fusion(c, cfg, cm) -> (fused Circuit, FusionStats dict)."""
    cfg = cfg or FusionConfig()
    h = _vp()
    st = _FusionStatsC()
    cc = cfg._c()
    _check(_lib.tsc_run_fusion(c._h, C.byref(cc), cost_model._h if cost_model else None, C.byref(h), C.byref(st)))
    stats = {f: getattr(st, f) for f, _ in _FusionStatsC._fields_}
    return Circuit(_handle=h.value), stats


# ================================================================ device ===
class Context:
    """One B200 (tsg_ctx).  Raises SimError when no CUDA device is present."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(_lib.tsg_ctx_create(device, C.byref(h)))
        self._h = h.value
        self.device = device
        sms = C.c_int()
        _check(_lib.tsg_ctx_info(self._h, None, C.byref(sms)))
        self.num_sms = sms.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsg_ctx_destroy(self._h)
            self._h = None


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class Statevector:
    """Device-resident SoA statevector; precision 'f64' | 'f32'."""

    def __init__(self, n: int, precision: str = "f64", ctx: Context | None = None):
        self.ctx = ctx or default_context()
        bits = {"f64": 64, "f32": 32, "c128": 64, "c64": 32}[precision]
        h = _vp()
        _check(_lib.tsg_state_create(self.ctx._h, n, bits, C.byref(h)))
        self._h = h.value
        self.n = n
        self.precision_bits = bits

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsg_state_destroy(self._h)
            self._h = None

    def init_zero(self):
        _check(_lib.tsg_state_init_zero(self._h))
        return self

    def init_basis(self, index: int):
        _check(_lib.tsg_state_init_basis(self._h, index))
        return self

    def init_random(self, seed: int):
        _check(_lib.tsg_state_init_random(self._h, seed))
        return self

    def upload(self, re: np.ndarray, im: np.ndarray):
        re = np.ascontiguousarray(re, dtype=np.float64)
        im = np.ascontiguousarray(im, dtype=np.float64)
        if re.size != 1 << self.n or im.size != 1 << self.n:
            raise ConfigError("host arrays must have 2^n entries")
        _check(_lib.tsg_state_upload(self._h, re.ctypes.data_as(_dp), im.ctypes.data_as(_dp)))
        return self

    def upload_range(self, begin: int, re: np.ndarray, im: np.ndarray):
        """Overwrite amplitudes [begin, begin + len(re)) from host arrays."""
        re = np.ascontiguousarray(re, dtype=np.float64).reshape(-1)
        im = np.ascontiguousarray(im, dtype=np.float64).reshape(-1)
        if re.size != im.size:
            raise ConfigError("re and im must have the same length")
        _check(_lib.tsg_state_upload_range(self._h, begin, re.size, re.ctypes.data_as(_dp), im.ctypes.data_as(_dp)))
        return self

    def download(self, begin: int = 0, count: int | None = None):
        count = (1 << self.n) - begin if count is None else count
        re = np.empty(count)
        im = np.empty(count)
        _check(_lib.tsg_state_download_range(self._h, begin, count, re.ctypes.data_as(_dp), im.ctypes.data_as(_dp)))
        return re, im

    def gather(self, indices):
        """Amplitudes at arbitrary indices (one device gather, one copy back) -> (re, im)."""
        idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
        re = np.empty(idx.size)
        im = np.empty(idx.size)
        _check(_lib.tsg_state_gather(self._h, idx.ctypes.data_as(C.POINTER(_u64)), idx.size,
                                     re.ctypes.data_as(_dp), im.ctypes.data_as(_dp)))
        return re, im

    def amplitudes(self) -> np.ndarray:
        re, im = self.download()
        return re + 1j * im

    def dump(self, path: str):
        """QSV1 amplitude dump."""
        _check(_lib.tsg_state_dump(self._h, os.fsencode(path)))
        return self

    def load(self, path: str):
        """Load a QSV1 dump of the same precision and qubit count."""
        _check(_lib.tsg_state_load(self._h, os.fsencode(path)))
        return self

    def synchronize(self):
        _check(_lib.tsg_synchronize(self._h))

    def timer_begin(self):
        _check(_lib.tsg_timer_begin(self._h))

    def timer_end(self) -> float:
        out = C.c_double()
        _check(_lib.tsg_timer_end(self._h, C.byref(out)))
        return out.value

    def norm(self) -> float:
        out = C.c_double()
        _check(_lib.tsg_norm(self._h, C.byref(out)))
        return out.value

    def copy_from(self, other: "Statevector"):
        _check(_lib.tsg_state_copy(self._h, other._h))
        return self


def init_zero_state(n: int, precision: str = "f64") -> Statevector:
    return Statevector(n, precision).init_zero()


def norm(sv: Statevector) -> float:
    return sv.norm()


def compare_states(a: Statevector, b) -> float:
    """max_i |a_i - b_i| against another Statevector or host (re, im) arrays."""
    out = C.c_double()
    if isinstance(b, Statevector):
        _check(_lib.tsg_compare_states(a._h, b._h, C.byref(out)))
    else:
        re = np.ascontiguousarray(b[0], dtype=np.float64)
        im = np.ascontiguousarray(b[1], dtype=np.float64)
        _check(_lib.tsg_compare(a._h, re.ctypes.data_as(_dp), im.ctypes.data_as(_dp), C.byref(out)))
    return out.value


def overlap(a: Statevector, b: Statevector) -> complex:
    re, im = C.c_double(), C.c_double()
    _check(_lib.tsg_overlap(a._h, b._h, C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


class KernelPlan:
    """plan_kernel(g, n, s=0, zero_tol, one_tol, runtime_matrix)."""

    def __init__(self, gate: Gate, n: int, zero_tol=1e-8, one_tol=1e-8, runtime_matrix=False, ctx=None):
        self.ctx = ctx or _default_ctx
        m = _matrix_arg(gate.matrix)
        h = _vp()
        _check(_lib.tsg_plan_create(self.ctx._h if self.ctx else None, n, gate.k, _ints(gate.targets),
                                    m.ctypes.data_as(_dp), zero_tol, one_tol, int(runtime_matrix), C.byref(h)))
        self._h = h.value
        self.gate = gate
        self.n = n
        self.runtime_matrix = runtime_matrix

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsg_plan_destroy(self._h)
            self._h = None

    def info(self) -> dict:
        pi = PlanInfo()
        _check(_lib.tsg_plan_info_get(self._h, C.byref(pi)))
        return _plan_info_dict(pi)


def plan_kernel(gate: Gate, n: int, s: int = 0, zero_tol=1e-8, one_tol=1e-8, runtime_matrix=False) -> KernelPlan:
    if s != 0:
        raise ConfigError("the B200 kernels use the GPU ABI's s = 0 loop (PAPER.md:380)")
    return KernelPlan(gate, n, zero_tol, one_tol, runtime_matrix)


def apply_kernel(plan: KernelPlan, sv: Statevector, matrix_override=None, t_begin: int = 0, t_end: int | None = None):
    """apply_kernel(plan, state, override, t_begin, t_end) over s = 0 groups."""
    ov = None
    if matrix_override is not None:
        arr = _matrix_arg(matrix_override)
        ov = arr.ctypes.data_as(_dp)
    _check(_lib.tsg_apply(sv._h, plan._h, ov, t_begin, (1 << 64) - 1 if t_end is None else t_end))


class Program:
    """A fused circuit planned once and replayed (CUDA graph) -- run_circuit's engine."""

    def __init__(self, fused: Circuit, precision: str = "f64", zero_tol=1e-8, one_tol=1e-8, ctx=None):
        self.ctx = ctx or default_context()
        bits = {"f64": 64, "f32": 32, "c128": 64, "c64": 32}[precision]
        h = _vp()
        _check(_lib.tsg_program_create(self.ctx._h, fused._h, zero_tol, one_tol, bits, C.byref(h)))
        self._h = h.value
        self.n_gates = len(fused)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsg_program_destroy(self._h)
            self._h = None

    def run(self, sv: Statevector, use_graph: bool = True) -> dict:
        r = RunReport()
        _check(_lib.tsg_program_run(sv._h, self._h, int(use_graph), C.byref(r)))
        return r.as_dict()

    def enqueue(self, sv: Statevector, use_graph: bool = True) -> None:
        """Asynchronous run on the state's stream (time it with sv.timer_begin/end)."""
        _check(_lib.tsg_program_enqueue(sv._h, self._h, int(use_graph)))

    def run_profiled(self, sv: Statevector):
        secs = np.zeros(max(1, self.n_gates))
        r = RunReport()
        _check(_lib.tsg_program_run_profiled(sv._h, self._h, secs.ctypes.data_as(_dp), C.byref(r)))
        return secs[: self.n_gates], r.as_dict()

    def steps(self) -> list:
        """Launch steps in order: {kind, first_gate, n_gates, high, kernel} (tsg_program_step_info)."""
        cnt = _u64()
        _check(_lib.tsg_program_step_count(self._h, C.byref(cnt)))
        out = []
        for i in range(cnt.value):
            si = StepInfo()
            _check(_lib.tsg_program_step_info(self._h, i, C.byref(si)))
            out.append({"kind": STEP_KINDS[si.kind], "first_gate": si.first_gate, "n_gates": si.n_gates,
                        "high": list(si.high[:si.n_high]), "kernel": si.kernel.decode()})
        return out

    def pass_layouts(self) -> list:
        """Per step: (register layouts loaded through shared memory, layouts reached
        with warp shuffles) -- (0, 0) for steps that are not tile passes."""
        cnt = _u64()
        _check(_lib.tsg_program_step_count(self._h, C.byref(cnt)))
        out = []
        for i in range(cnt.value):
            a, b = C.c_int(), C.c_int()
            _check(_lib.tsg_program_pass_layouts(self._h, i, C.byref(a), C.byref(b)))
            out.append((a.value, b.value))
        return out

    def jit_kernels(self) -> dict:
        """JIT-compiled kernels the program runs: {"passes": tile passes, "gates":
        standalone launches with a JIT DMMA product}."""
        a, b = C.c_int(), C.c_int()
        _check(_lib.tsg_program_jit_kernels(self._h, C.byref(a), C.byref(b)))
        return {"passes": a.value, "gates": b.value}

    def gate_info(self, i: int) -> dict:
        pi = PlanInfo()
        _check(_lib.tsg_program_gate_info(self._h, i, C.byref(pi)))
        return _plan_info_dict(pi)


def plan_passes(fused: Circuit, precision: str = "f64", zero_tol=1e-8, one_tol=1e-8) -> list:
    """Host-only tile-pass grouping (tilesim/pass.hpp) exactly as Program builds it:
    a list of steps {"gates": [...], "is_pass": bool, "is_permute": bool, "high": [...]}
    in launch order (is_permute: a run of qubit-permutation gates, one k_permute step)."""
    bits = {"f64": 64, "f32": 32, "c128": 64, "c64": 32}[precision]
    g = max(1, len(fused))
    sog = np.zeros(g, dtype=np.int32)
    isp = np.zeros(g, dtype=np.int32)
    high = np.zeros(16 * g, dtype=np.int32)
    ns = _u64()
    _check(_lib.tsc_plan_passes(fused._h, bits, zero_tol, one_tol, sog.ctypes.data_as(_ip), isp.ctypes.data_as(_ip),
                                high.ctypes.data_as(_ip), C.byref(ns)))
    steps = [{"gates": [], "is_pass": bool(isp[s] == 1), "is_permute": bool(isp[s] == 2),
              "high": [int(h) for h in high[16 * s:16 * s + 16] if h >= 0]} for s in range(ns.value)]
    for gi in range(len(fused)):
        if sog[gi] >= 0:
            steps[sog[gi]]["gates"].append(gi)
    return steps


_sig("tsc_pass_jit_precompile", [_vp, C.c_int, C.c_double, C.c_double, _ip])


def pass_jit_precompile(fused: Circuit, precision: str = "f64", zero_tol=1e-8, one_tol=1e-8) -> int:
    """NVRTC-compile the JIT tile passes a Program of `fused` would use into the
    JIT disk cache (host only); returns the program's pass count."""
    n = C.c_int()
    _check(_lib.tsc_pass_jit_precompile(fused._h, 64 if precision in ("f64", "c128") else 32, zero_tol, one_tol,
                                        C.byref(n)))
    return n.value


def run_circuit(c: Circuit, sv: Statevector, zero_tol=1e-8, one_tol=1e-8, use_graph=True) -> dict:
    """run_circuit: plan every gate, apply in order on the device."""
    prec = "f64" if sv.precision_bits == 64 else "f32"
    prog = Program(c, prec, zero_tol, one_tol, sv.ctx)
    return prog.run(sv, use_graph)


def bench_cost_model(bench_n: int = 28, k_max: int = 6, precision: str = "f64", repetitions: int = 5,
                     seed: int = 1, ctx: Context | None = None, sm_counts=None) -> CostModel:
    """GPU bench_cost_model.  `threads` of the records = SMs
    the kernels span: the full device by default, or each of sm_counts."""
    ctx = ctx or default_context()
    h = _vp()
    bits = 64 if precision in ("f64", "c128") else 32
    if sm_counts is None:
        _check(_lib.tsg_bench_cost_model(ctx._h, bench_n, k_max, bits, repetitions, seed, C.byref(h)))
    else:
        _check(_lib.tsg_bench_cost_model_sms(ctx._h, bench_n, k_max, bits, repetitions, seed, _ints(sm_counts),
                                             len(sm_counts), C.byref(h)))
    return CostModel(_handle=h.value)


# ============================================================== sharding ===
_sig("tsc_shard_plan_create", [_vp, C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(_vp)])
_sig("tsc_shard_plan_stats", [_vp, C.POINTER(_u64), C.POINTER(_u64), _ip])
_sig("tsc_shard_plan_destroy", [_vp])
_sig("tsc_shard_plan_info", [_vp, _ip, _ip, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)])
_sig("tsc_shard_plan_op", [_vp, _u64, _ip, _ip, _ip, _dp, _ip, _ip, _ip, _ip, _ip])
_sig("tsc_shard_rank_subgate", [_vp, _u64, _u64, _ip, _ip, _dp])
_sig("tsc_shard_final_pos", [_vp, _ip])
_sig("tsg_vshard_run", [_vp, _vp, C.c_int, _dp, _dp, _dp, _dp, C.POINTER(RunReport)])
_sig("tsg_dist_unique_id", [C.POINTER(C.c_ubyte)])
_sig("tsg_dist_create", [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_ubyte), C.POINTER(_vp)])
_sig("tsg_dist_destroy", [_vp])
_sig("tsg_dist_init_basis", [_vp, _u64])
_sig("tsg_dist_run", [_vp, _vp, C.POINTER(RunReport)])
_sig("tsg_dist_run_local_only", [_vp, _vp, C.POINTER(RunReport)])
_sig("tsg_dist_upload_local", [_vp, _dp, _dp])
_sig("tsg_dist_dump", [_vp, C.c_char_p, _ip])
_sig("tsg_dist_load", [_vp, C.c_char_p, _ip])
_sig("tsg_rendezvous_selftest", [C.POINTER(C.c_ubyte), C.c_int, C.c_int, C.c_int, C.POINTER(_u64)])
_sig("tsg_dist_download_local", [_vp, _dp, _dp])
_sig("tsg_dist_local_sumsq", [_vp, _dp])

SHARD_KINDS = ("local", "rank_block", "swap")


class ShardPlan:
    """Global-qubit sharding of a fused circuit over 2^n_global ranks (tilesim/shard.hpp)."""

    def __init__(self, fused: Circuit, n_global: int, zero_tol=1e-8, one_tol=1e-8, pipeline_bits: int = 2):
        h = _vp()
        _check(_lib.tsc_shard_plan_create(fused._h, n_global, zero_tol, one_tol, pipeline_bits, C.byref(h)))
        self._h = h.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsc_shard_plan_destroy(self._h)
            self._h = None

    def info(self) -> dict:
        n, g = C.c_int(), C.c_int()
        ops, sw, rb = _u64(), _u64(), _u64()
        _check(_lib.tsc_shard_plan_info(self._h, C.byref(n), C.byref(g), C.byref(ops), C.byref(sw), C.byref(rb)))
        xo, pp, pb = _u64(), _u64(), C.c_int()
        _check(_lib.tsc_shard_plan_stats(self._h, C.byref(xo), C.byref(pp), C.byref(pb)))
        return {"n": n.value, "n_global": g.value, "n_local": n.value - g.value, "ops": ops.value,
                "swaps": sw.value, "rank_blocks": rb.value, "exchanges": xo.value, "pipelined_exchanges": pp.value,
                "pipeline_bits": pb.value}

    def op(self, i: int) -> dict:
        kind, k, ns, src, pb, po = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        t = (C.c_int * 12)()
        m = np.zeros(2 * 4 ** 6)
        sp = (C.c_int * 64)()
        _check(_lib.tsc_shard_plan_op(self._h, i, C.byref(kind), C.byref(k), t, m.ctypes.data_as(_dp), C.byref(ns),
                                      sp, C.byref(src), C.byref(pb), C.byref(po)))
        gate = None
        if kind.value != 2:
            d = 1 << k.value
            gate = Gate(list(t)[: k.value], m[: 2 * d * d].view(np.complex128).reshape(d, d).copy())
        return {"kind": SHARD_KINDS[kind.value], "gate": gate, "source_gate": src.value,
                "swaps": [(sp[2 * s], sp[2 * s + 1]) for s in range(ns.value)], "pipeline_bits": pb.value,
                "pipeline_ops": po.value}

    def ops(self):
        return [self.op(i) for i in range(self.info()["ops"])]

    def rank_subgate(self, i: int, rank: int) -> Gate:
        k = C.c_int()
        t = (C.c_int * 12)()
        m = np.zeros(2 * 4 ** 6)
        _check(_lib.tsc_shard_rank_subgate(self._h, i, rank, C.byref(k), t, m.ctypes.data_as(_dp)))
        d = 1 << k.value
        return Gate(list(t)[: k.value], m[: 2 * d * d].view(np.complex128).reshape(d, d).copy())

    def final_pos(self):
        info = self.info()
        pos = (C.c_int * info["n"])()
        _check(_lib.tsc_shard_final_pos(self._h, pos))
        return list(pos)


def physical_permutation(final_pos, n: int) -> np.ndarray:
    """phys[x] = physical index of logical basis state x under final_pos."""
    x = np.arange(1 << n, dtype=np.uint64)
    phys = np.zeros(1 << n, dtype=np.uint64)
    for q, p in enumerate(final_pos):
        phys |= ((x >> np.uint64(q)) & np.uint64(1)) << np.uint64(p)
    return phys


def vshard_run(plan: ShardPlan, re: np.ndarray, im: np.ndarray, precision: str = "f64", ctx: Context | None = None):
    """Run a shard plan on 2^n_global virtual shards of ONE device (single-GPU
    emulation of the distributed path).  Inputs/outputs: full state, logical order."""
    ctx = ctx or default_context()
    re = np.ascontiguousarray(re, dtype=np.float64)
    im = np.ascontiguousarray(im, dtype=np.float64)
    ore, oim = np.empty_like(re), np.empty_like(im)
    r = RunReport()
    _check(_lib.tsg_vshard_run(ctx._h, plan._h, 64 if precision in ("f64", "c128") else 32, re.ctypes.data_as(_dp),
                               im.ctypes.data_as(_dp), ore.ctypes.data_as(_dp), oim.ctypes.data_as(_dp), C.byref(r)))
    return ore, oim, r.as_dict()


class DistState:
    """This rank's shard of a 2^n statevector over 2^n_global processes of one
    box: shards exported over CUDA IPC, exchanges as in-place peer-memory
    kernels (tsg_dist_*).  Creation, run and close are collective."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(_lib.tsg_dist_unique_id(buf))
        return bytes(buf)

    def __init__(self, n: int, n_global: int, rank: int, uid: bytes, precision: str = "f64",
                 ctx: Context | None = None):
        self.ctx = ctx or default_context()
        buf = (C.c_ubyte * 128)(*uid)
        h = _vp()
        _check(_lib.tsg_dist_create(self.ctx._h, n, 64 if precision in ("f64", "c128") else 32, n_global, rank, buf,
                                    C.byref(h)))
        self._h = h.value
        self.n, self.n_global, self.rank = n, n_global, rank

    def close(self):
        """Collective teardown (every rank must call it)."""
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tsg_dist_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def init_basis(self, x: int):
        _check(_lib.tsg_dist_init_basis(self._h, x))
        return self

    def upload_local(self, re: np.ndarray, im: np.ndarray):
        re = np.ascontiguousarray(re, dtype=np.float64)
        im = np.ascontiguousarray(im, dtype=np.float64)
        if re.size != 1 << (self.n - self.n_global) or im.size != re.size:
            raise ConfigError("host arrays must have 2^(n - n_global) entries")
        _check(_lib.tsg_dist_upload_local(self._h, re.ctypes.data_as(_dp), im.ctypes.data_as(_dp)))
        return self

    def run(self, plan: ShardPlan) -> dict:
        r = RunReport()
        _check(_lib.tsg_dist_run(self._h, plan._h, C.byref(r)))
        return r.as_dict()

    def run_local_only(self, plan: ShardPlan) -> dict:
        """The plan's local segments alone (compute-only timeline; state meaningless afterwards)."""
        r = RunReport()
        _check(_lib.tsg_dist_run_local_only(self._h, plan._h, C.byref(r)))
        return r.as_dict()

    def download_local(self):
        m = 1 << (self.n - self.n_global)
        re, im = np.empty(m), np.empty(m)
        _check(_lib.tsg_dist_download_local(self._h, re.ctypes.data_as(_dp), im.ctypes.data_as(_dp)))
        return re, im

    def local_sumsq(self) -> float:
        out = C.c_double()
        _check(_lib.tsg_dist_local_sumsq(self._h, C.byref(out)))
        return out.value

    def dump(self, path: str, final_pos) -> None:
        """Sharded QSV1: this rank's shard to <path>.r<rank>, the layout (rank 0) to <path>.layout."""
        _check(_lib.tsg_dist_dump(self._h, os.fsencode(path), _ints(list(final_pos))))

    def load(self, path: str) -> list:
        """Read this rank's shard of a sharded QSV1 dump; returns the qubit map it is laid out in."""
        pos = (C.c_int * self.n)()
        _check(_lib.tsg_dist_load(self._h, os.fsencode(path), pos))
        return list(pos)


def rendezvous_selftest(uid: bytes, rank: int, world: int, iters: int = 100) -> int:
    """Host-only exercise of the ranks' shared-memory rendezvous (no device)."""
    buf = (C.c_ubyte * 128)(*uid)
    out = _u64()
    _check(_lib.tsg_rendezvous_selftest(buf, rank, world, iters, C.byref(out)))
    return out.value
