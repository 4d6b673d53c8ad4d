"""Numerics of the complex64 sub-gate kernels: one dense random gate per case
on a 16-qubit state, against numpy complex128 of the same (rounded) input.
Run once with TSG_UMMA=0 (FP64-widened DMMA) and once without (tcgen05)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

n = int(os.environ.get('UC_N', '16'))
cases = [[0, 1, 2], [5, 6, 7], [10, 12, 15], [0, 1, 2, 3], [6, 7, 8, 9], [1, 5, 9, 13], [12, 13, 14, 15],
         [0, 1, 2, 3, 4], [5, 6, 7, 8, 9], [0, 3, 7, 11, 15], [11, 12, 13, 14, 15]]
rng = np.random.default_rng(7)
psi0 = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(np.complex64)
psi0 /= np.linalg.norm(psi0)
for t in cases:
    k = len(t)
    m = random_gate_matrix(k, 100 + sum(t), "dense")
    c = ts.Circuit(n)
    c.add_matrix(t, m)
    prog = ts.Program(c, "f32")
    sv = ts.Statevector(n, "f32").upload(psi0.real.astype(np.float64), psi0.imag.astype(np.float64))
    prog.run(sv)
    got = sv.amplitudes()
    # exact: apply m on targets t (bit b of the matrix index = qubit t[b])
    x = psi0.astype(np.complex128).reshape([2] * n)  # axis i = qubit n-1-i
    axes = [n - 1 - q for q in reversed(t)]  # matrix index msb first
    xm = np.moveaxis(x, axes, list(range(k))).reshape(1 << k, -1)
    y = (m @ xm).reshape([2] * k + [2] * (n - k))
    want = np.moveaxis(y, list(range(k)), axes).reshape(-1)
    err = np.abs(got - want).max()
    dn = np.vdot(got, got).real - np.vdot(want, want).real
    print(f"targets={t} kernel={prog.steps()[0]['kernel']} max|d|={err:.3e} rel={err / np.abs(want).max():.3e} "
          f"d|psi|^2={dn:+.2e}")
