"""Dense 6-qubit gates at n = 30 on several target sets (device time per
gate, median of 6): complex128 on k_stream_dmma<ks=6> (or k_tile with
TSG_NO_DMMA6=1 in the environment of a build that honours it), complex64 on
k_stream_umma<ks=6>.  usage: d6_bench.py [f64|f32] [VARIANT_ROOT]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2:  # a variant build's root (scripts/build_variant.sh)
    sys.path.insert(0, sys.argv[2])
import paper_2503_19894_b200 as ts  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
n = 30
sweep = 2 * (1 << n) * (16 if prec == "f64" else 8) / 6549.4e9 * 1e3
sv = ts.Statevector(n, prec).init_random(1)
os.environ["TSG_NO_BLOCK_SPLIT"] = "1"
for t in ([0, 1, 2, 3, 4, 5], [3, 4, 5, 6, 7, 8], [6, 7, 8, 9, 10, 11], [12, 13, 14, 15, 16, 17],
          [24, 25, 26, 27, 28, 29], [2, 7, 13, 19, 22, 28]):
    c = ts.Circuit(n)
    for i in range(6):
        c.add_matrix(t, random_gate_matrix(6, 20 + i, "dense"))
    prog = ts.Program(c, prec)
    prog.run(sv)
    secs, _ = prog.run_profiled(sv)
    ms = sorted(secs)[len(secs) // 2] * 1e3
    print(f"targets={t} {prog.steps()[0]['kernel']:22s} {ms:7.3f} ms  ({sweep / ms:.2f} of an HBM sweep)")
