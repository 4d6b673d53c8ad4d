"""Device time of one dense k-qubit complex64 gate at n = 30 for several
target sets (run_profiled events).  usage: umma_bench.py [N] [KS...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("PB_ROOT"):  # a variant build (A/B)
    sys.path.insert(0, os.environ["PB_ROOT"])
import paper_2503_19894_b200 as ts  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
kss = [int(x) for x in sys.argv[2:]] or [3, 4, 5]
sets = {3: [[0, 1, 2], [3, 4, 5], [8, 9, 10], [20, 25, 29], [2, 9, 17]],
        4: [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11], [26, 27, 28, 29], [1, 9, 17, 25], [2, 3, 4, 5], [1, 2, 3, 4]],
        5: [[0, 1, 2, 3, 4], [5, 6, 7, 8, 9], [10, 11, 12, 13, 14], [25, 26, 27, 28, 29], [0, 7, 14, 21, 28],
            [1, 2, 3, 4, 5], [3, 7, 10, 12, 15]]}
sv = ts.Statevector(n, "f32").init_zero()
bytes_ = 2 * 8 * (1 << n)
for ks in kss:
    for t in sets[ks]:
        c = ts.Circuit(n)
        for _ in range(8):
            c.add_matrix(t, random_gate_matrix(ks, 3, "dense"))
        prog = ts.Program(c, "f32")
        prog.run(sv)
        secs, _ = prog.run_profiled(sv)
        ms = sorted(secs)[len(secs) // 2] * 1e3
        print(f"ks={ks} targets={t} {prog.steps()[0]['kernel']:22s} {ms:7.3f} ms  {bytes_ / ms / 1e6:7.1f} GB/s")
