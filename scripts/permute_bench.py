"""Device time of one qubit-permutation step at n qubits: bit reversal, a
15-cycle (two sweeps), and a high-only permutation.  usage: permute_bench.py [N] [PREC]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
amp = 16 if prec == "f64" else 8
cases = {"bitrev": [(i, n - 1 - i) for i in range(n // 2)],
         "lowhigh": [(i, i + 20) for i in range(5)],
         "cycle": [(i, i + 1) for i in range(14)],
         "high": [(10, 29), (11, 28), (12, 27), (13, 26)]}
sv = ts.Statevector(n, prec).init_zero()
for name, pairs in cases.items():
    c = ts.Circuit(n)
    for a, b in pairs:
        c.add("swap", [a, b])
    prog = ts.Program(c, prec)
    prog.run(sv)
    ts_ = []
    for _ in range(3):
        secs, rep = prog.run_profiled(sv)
        ts_.append(rep["execution_s"])
    t = min(ts_)
    sweeps = 2 if any("x2" in s["kernel"] for s in prog.steps()) else 1
    print(f"{name:8s} {[s['kernel'] for s in prog.steps()]} {t * 1e3:7.3f} ms  "
          f"{sweeps * 2 * amp * (1 << n) / t / 1e9:7.1f} GB/s")
