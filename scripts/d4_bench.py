"""Dense 4-qubit complex128 gates at n = 30 on several target sets (device
time per gate), for kernel-variant builds.  usage: d4_bench.py [REPO_ROOT]"""
import os
import sys

root = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import paper_2503_19894_b200 as ts  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests._util import random_gate_matrix  # noqa: E402

n = 30
sv = ts.Statevector(n, "f64").init_zero()
tot = 0.0
for t in ([0, 1, 2, 3], [2, 3, 4, 5], [4, 5, 6, 7], [7, 8, 9, 10], [13, 14, 15, 16], [26, 27, 28, 29], [1, 9, 17, 25]):
    c = ts.Circuit(n)
    for i in range(6):
        c.add_matrix(t, random_gate_matrix(4, 10 + i, "dense"))
    prog = ts.Program(c, "f64")
    prog.run(sv)
    secs, _ = prog.run_profiled(sv)
    ms = sorted(secs)[len(secs) // 2] * 1e3
    tot += ms
    print(f"targets={t} {prog.steps()[0]['kernel']:22s} {ms:7.3f} ms")
print(f"sum {tot:.3f} ms")
