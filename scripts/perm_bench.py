"""k_permute device time: QFT-30's bit-reversal step and two other involutions
at n = 30, complex128 and complex64 (PB_ROOT=<variant dir> for A/B; design
measurement), plus a parity check of each against numpy at n = 16."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("PB_ROOT"):
    sys.path.insert(0, os.environ["PB_ROOT"])
import paper_2503_19894_b200 as ts  # noqa: E402

print("library", ts._lib._name if hasattr(ts, "_lib") else "?")


def swaps_circuit(n, pairs):
    c = ts.Circuit(n)
    for a, b in pairs:
        c.add("swap", [a, b])
    return c


for n, prec in ((30, "f64"), (30, "f32")):
    sv = ts.Statevector(n, prec).init_basis(5)
    for name, pairs in (("bitrev", [(i, n - 1 - i) for i in range(n // 2)]), ("low-high", [(0, 29), (1, 28), (2, 27)]),
                        ("mid", [(5, 20), (6, 21), (12, 13)])):
        prog = ts.Program(swaps_circuit(n, pairs), prec)
        prog.run(sv)
        best = min(prog.run(sv)["execution_s"] for _ in range(5))
        print(f"{prec} {name:9s} {[s['kernel'] for s in prog.steps()]} {best * 1e3:7.3f} ms")
n = 16
rng = np.random.default_rng(3)
psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
for pairs in ([(i, n - 1 - i) for i in range(n // 2)], [(0, 15), (1, 14), (2, 13)], [(5, 10), (6, 11), (7, 8)]):
    sv = ts.Statevector(n, "f64").upload(psi.real.copy(), psi.imag.copy())
    ts.Program(swaps_circuit(n, pairs), "f64").run(sv)
    perm = list(range(n))
    for a, b in pairs:
        perm[a], perm[b] = perm[b], perm[a]
    idx = np.arange(1 << n)
    src = np.zeros_like(idx)
    for q in range(n):
        src |= ((idx >> q) & 1) << perm[q]
    want = psi[src]
    print("parity", pairs[:2], float(np.abs(sv.amplitudes() - want).max()))
