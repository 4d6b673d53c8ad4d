"""k_stream_umma: complex64 4- and 5-qubit sub-gates on the INT8 tensor cores
(kernels_umma.cuh, INT8 slices with exact INT32 accumulation).

Checks each geometry the kernel takes (high and scattered targets, controls
folded into the run or the tile base) against numpy complex128 of the same
rounded input, the SPEC complex64 bar against the CPU oracle, and that the
result carries no bias: a TF32 3-split, whose FP32 tensor-core accumulation
truncates, lost ~2e-7 of the norm per gate; the INT8 slices must not drift.
"""
import numpy as np
import pytest

import paper_2503_19894_b200 as ts
from oracle import binding as ob
from tests._util import random_gate_matrix, to_oracle

pytestmark = pytest.mark.gpu


def _apply_numpy(psi, targets, m):
    """m on `targets` (bit b of the matrix index = qubit targets[b])."""
    n = int(np.log2(psi.size))
    k = len(targets)
    x = psi.astype(np.complex128).reshape([2] * n)  # axis i = qubit n-1-i
    axes = [n - 1 - q for q in reversed(targets)]
    xm = np.moveaxis(x, axes, list(range(k))).reshape(1 << k, -1)
    y = (m @ xm).reshape([2] * k + [2] * (n - k))
    return np.moveaxis(y, list(range(k)), axes).reshape(-1)


def _state(n, seed):
    rng = np.random.default_rng(seed)
    psi = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(np.complex64)
    return psi / np.linalg.norm(psi)


@pytest.mark.parametrize("targets,kind", [
    ([4, 5, 6, 7], "dense"), ([1, 5, 9, 13], "dense"), ([12, 13, 14, 15], "dense"), ([2, 3, 11, 12], "dense"),
    ([5, 6, 7, 8, 9], "dense"), ([3, 7, 10, 12, 15], "dense"), ([11, 12, 13, 14, 15], "dense"),
    ([2, 6, 7, 8, 9], "controlled"), ([3, 4, 5, 9, 14, 15], "controlled"), ([1, 2, 3, 4, 5, 6], "controlled"),
    ([2, 3, 4, 5], "dense"), ([1, 2, 3, 4], "dense"), ([1, 2, 3, 4, 5], "dense"),  # chunked stage (low targets)
    ([0, 7, 11, 15], "dense"), ([0, 6, 9, 12, 14], "dense"),  # bit-0 target, lanes nearly contiguous
    ([6, 7, 8, 9, 10, 11], "dense"), ([2, 5, 7, 9, 12, 15], "dense"), ([3, 4, 5, 6, 7, 8], "perm"),  # 6 qubits
    ([1, 4, 6, 8, 10, 13, 15], "controlled"), ([0, 1, 2, 3, 4, 5], "dense"),  # 6 qubits from bit 0 (chunked)
])
def test_umma_gate_matches_numpy(targets, kind):
    n = 16
    m = random_gate_matrix(len(targets), 31 + sum(targets), kind)
    c = ts.Circuit(n)
    c.add_matrix(targets, m)
    prog = ts.Program(c, "f32")
    kernels = [s["kernel"] for s in prog.steps()]
    assert any(k.startswith("k_stream_umma") for k in kernels), kernels
    psi0 = _state(n, 5)
    sv = ts.Statevector(n, "f32").upload(psi0.real.astype(np.float64), psi0.imag.astype(np.float64))
    prog.run(sv)
    want = _apply_numpy(psi0, targets, m)
    err = np.abs(sv.amplitudes() - want).max()
    # three 7-bit slices per operand: ~2^-21 of each group row's scale
    assert err <= 4e-6 * np.abs(want).max(), err
    # SPEC complex64 bar against the CPU oracle
    ore, oim = psi0.real.copy(), psi0.imag.copy()
    ob.run_circuit(to_oracle(c), ore, oim)
    assert ts.compare_states(sv, (ore.astype(np.float64), oim.astype(np.float64))) <= 1e-5


def test_umma_norm_does_not_drift():
    """60 dense 4- and 5-qubit gates: unitary, so the norm must stay 1 up to
    unbiased rounding (a truncating accumulator loses ~1e-5 here)."""
    n = 17
    rng = np.random.default_rng(9)
    c = ts.Circuit(n)
    for i in range(60):
        k = 4 + i % 2
        t = sorted(int(q) for q in rng.choice(np.arange(1, n), size=k, replace=False))
        c.add_matrix(t, random_gate_matrix(k, 500 + i, "dense"))
    prog = ts.Program(c, "f32")
    assert sum(s["kernel"].startswith("k_stream_umma") for s in prog.steps()) >= 50
    psi0 = _state(n, 6)
    sv = ts.Statevector(n, "f32").upload(psi0.real.astype(np.float64), psi0.imag.astype(np.float64))
    prog.run(sv)
    psi = sv.amplitudes()
    assert abs(np.vdot(psi, psi).real - 1.0) <= 2e-6
    want = psi0.astype(np.complex128)
    for g in [c.gate(i) for i in range(len(c))]:
        want = _apply_numpy(want, list(g.targets), np.asarray(g.matrix))
    # normalised fidelity at the north star's bar (the norm is checked above)
    fid = abs(np.vdot(want, psi)) ** 2 / (np.vdot(want, want).real * np.vdot(psi, psi).real)
    assert fid >= 1 - 1e-9, 1 - fid


def test_umma_bit0_geometry():
    """A target on qubit 0: the tensor-core kernel only when the lanes stay
    nearly contiguous (umma_plan); contiguous low targets keep the DMMA product."""
    c = ts.Circuit(14)
    c.add_matrix([0, 1, 2, 3], random_gate_matrix(4, 3, "dense"))
    prog = ts.Program(c, "f32")
    assert [s["kernel"] for s in prog.steps()] == ["k_stream_dmma<ks=4>"]
    c = ts.Circuit(16)
    c.add_matrix([0, 7, 11, 15], random_gate_matrix(4, 4, "dense"))
    prog = ts.Program(c, "f32")
    assert [s["kernel"] for s in prog.steps()] == ["k_stream_umma<ks=4>"]
