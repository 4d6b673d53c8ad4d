"""JIT-compiled tile passes (NVRTC, pass_jit.cu) against the interpreter.

A JIT pass runs the same device functions with the op table folded into
constants, so its results must equal the interpreter's bit for bit; both are
checked against the CPU oracle as well.  TSG_PASS_JIT_MIN_N=1 JIT-compiles
passes at test sizes (the default threshold is 24 qubits)."""
import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import to_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,depth,kmax,prec", [("qft", 16, 1, 5, "f64"), ("qft", 17, 1, 3, "f64"),
                                                    ("rqc", 16, 8, 4, "f64"), ("hes", 16, 4, 5, "f32"),
                                                    ("qaoa", 16, 4, 5, "f32"), ("iqp", 15, 4, 5, "f64"),
                                                    ("ala", 14, 4, 3, "f32")])
def test_jit_pass_equals_interpreter(kind, n, depth, kmax, prec, monkeypatch):
    monkeypatch.setenv("TSG_PASS_FORCE", "1")  # every eligible run of gates becomes a pass
    fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 3), ts.FusionConfig(k_max=kmax))
    monkeypatch.setenv("TSG_PASS_JIT_MIN_N", "1")
    pj = ts.Program(fused, prec)
    monkeypatch.setenv("TSG_PASS_JIT", "0")
    pi = ts.Program(fused, prec)
    kj = [s["kernel"] for s in pj.steps()]
    ki = [s["kernel"] for s in pi.steps()]
    assert "k_pass_jit" in kj and "k_pass_jit" not in ki, (kj, ki)
    a = ts.Statevector(n, prec).init_random(5)
    b = ts.Statevector(n, prec).copy_from(a)
    re0, im0 = a.download()
    pj.run(a)
    pi.run(b)
    assert ts.compare_states(a, b) == 0.0
    pj.run(a, use_graph=True)  # graph capture of a JIT launch
    pi.run(b, use_graph=True)
    assert ts.compare_states(a, b) == 0.0
    dt = np.float64 if prec == "f64" else np.float32
    ore, oim = re0.astype(dt), im0.astype(dt)
    o = to_oracle(fused)
    ob.run_circuit(o, ore, oim, threads=4)  # the circuit was applied twice
    ob.run_circuit(o, ore, oim, threads=4)
    assert ts.compare_states(a, (ore.astype(np.float64), oim.astype(np.float64))) <= (1e-10 if prec == "f64" else 1e-5)


def test_precompile_warms_the_cache(tmp_path, monkeypatch):
    monkeypatch.setenv("TSG_JIT_CACHE_DIR", str(tmp_path))
    monkeypatch.setenv("TSG_PASS_JIT_MIN_N", "1")
    fused, _ = ts.run_fusion(ts.gen_benchmark("qft", 14), ts.FusionConfig(k_max=4))
    n = ts.pass_jit_precompile(fused, "f64")
    assert n > 0 and len(list(tmp_path.glob("*.cubin"))) >= 1
    prog = ts.Program(fused, "f64")
    assert sum(s["kernel"] == "k_pass_jit" for s in prog.steps()) == n


@pytest.mark.parametrize("kind,n,depth,kmax,prec", [("qft", 18, 1, 5, "f64"), ("hes", 16, 4, 5, "f32"),
                                                    ("rqc", 16, 8, 5, "f64"), ("qaoa", 16, 4, 5, "f32")])
def test_shuffle_layouts(kind, n, depth, kmax, prec, monkeypatch):
    """Register layouts reached with warp shuffles (register <-> lane swaps)
    against every layout through shared memory (TSG_PASS_SHFL=0), the
    interpreter against the JIT with shuffles, and the oracle."""
    monkeypatch.setenv("TSG_PASS_FORCE", "1")
    monkeypatch.setenv("TSG_PASS_JIT_MIN_N", "1")
    fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 3), ts.FusionConfig(k_max=kmax))
    ps = ts.Program(fused, prec)
    monkeypatch.setenv("TSG_PASS_JIT", "0")
    pi = ts.Program(fused, prec)
    monkeypatch.setenv("TSG_PASS_SHFL", "0")
    p0 = ts.Program(fused, prec)
    lay_s, lay_0 = ps.pass_layouts(), p0.pass_layouts()
    assert sum(b for _, b in lay_s) > 0, lay_s  # some layouts are shuffles
    assert sum(b for _, b in lay_0) == 0
    # same layouts in all: a shuffle replaces a shared-memory change one for one
    assert [a + b for a, b in lay_s] == [a + b for a, b in lay_0]
    a = ts.Statevector(n, prec).init_random(8)
    b = ts.Statevector(n, prec).copy_from(a)
    c = ts.Statevector(n, prec).copy_from(a)
    re0, im0 = a.download()
    ps.run(a)
    pi.run(b)
    p0.run(c)
    assert ts.compare_states(a, b) == 0.0  # JIT == interpreter, both with shuffles
    bar = 1e-12 if prec == "f64" else 1e-6  # thread positions change the order of diagonal factors only
    assert ts.compare_states(a, c) <= bar
    dt = np.float64 if prec == "f64" else np.float32
    ore, oim = re0.astype(dt), im0.astype(dt)
    ob.run_circuit(to_oracle(fused), ore, oim, threads=4)
    assert ts.compare_states(a, (ore.astype(np.float64), oim.astype(np.float64))) <= (1e-10 if prec == "f64" else 1e-5)
