"""Device times of the kernels a design variant changes (PB_ROOT=<variant dir>):
dense and RQC-like 5-qubit complex128 gates at n=30, the RQC-30 and QFT-30
programs.  Design measurements, not product."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("PB_ROOT"):
    sys.path.insert(0, os.environ["PB_ROOT"])
import paper_2503_19894_b200 as ts  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

print("library", ts._lib._name if hasattr(ts, "_lib") else "?")
n = 30
sv = ts.Statevector(n, "f64").init_basis(3)
for tg in ([3, 9, 14, 20, 27], [0, 1, 2, 3, 4], [7, 8, 9, 10, 11], [20, 21, 22, 23, 24]):
    p = ts.KernelPlan(ts.Gate(tg, random_gate_matrix(5, 5, "dense")), n)
    ts.apply_kernel(p, sv)
    sv.synchronize()
    sv.timer_begin()
    for _ in range(5):
        ts.apply_kernel(p, sv)
    print(f"dense ks5 {tg}: {sv.timer_end() / 5 * 1e3:.3f} ms")
for kind, depth in (("rqc", 20), ("qft", 1)):
    f, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 42), ts.FusionConfig(k_max=5))
    prog = ts.Program(f, "f64")
    prog.run(sv)
    best = min(prog.run(sv)["execution_s"] for _ in range(3))
    print(f"{kind}-30: {best * 1e3:.2f} ms")
