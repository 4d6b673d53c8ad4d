"""Shared helpers: move circuits between the product and the oracle (tests only)."""
import numpy as np

import paper_2503_19894_b200 as ts
from oracle import binding as ob


def to_oracle(c: ts.Circuit) -> ob.Circuit:
    """Rebuild a product circuit gate-for-gate (sorted targets, same bits) in the oracle."""
    o = ob.Circuit(c.n_qubits)
    for g in c.gates():
        o.add_matrix(g.targets, g.matrix)
    return o


def circuits_equal(a: ts.Circuit, b: ob.Circuit) -> None:
    ga, gb = a.gates(), b.gates()
    assert len(ga) == len(gb), (len(ga), len(gb))
    for i, (x, y) in enumerate(zip(ga, gb)):
        assert x.targets == y[0], (i, x.targets, y[0])
        assert np.array_equal(x.matrix, y[1]), i


def random_state(n: int, seed: int, dtype=np.float64):
    rng = np.random.default_rng(seed)
    re = rng.standard_normal(1 << n)
    im = rng.standard_normal(1 << n)
    s = np.sqrt((re * re + im * im).sum())
    return (re / s).astype(dtype), (im / s).astype(dtype)


def random_gate_matrix(k: int, seed: int, kind: str = "dense") -> np.ndarray:
    """dense: Haar-like unitary; sparse: random permutation with phases;
    diag: random phases; controlled: I (+) U on the top bit."""
    rng = np.random.default_rng(seed)
    d = 1 << k
    if kind == "dense":
        return ob.random_unitary(k, seed)
    if kind == "diag":
        return np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, d)))
    if kind == "perm":
        p = rng.permutation(d)
        m = np.zeros((d, d), complex)
        m[p, np.arange(d)] = np.exp(1j * rng.uniform(0, 2 * np.pi, d))
        return m
    if kind == "controlled":
        m = np.eye(d, dtype=complex)
        h = d // 2
        m[h:, h:] = ob.random_unitary(k - 1, seed) if k > 1 else np.exp(1j * 0.3)
        return m
    raise ValueError(kind)


def block_gate(mixed, block, seed: int):
    """A gate on sorted(mixed + block) that is block-diagonal in the `block`
    qubits, with an independent dense unitary on the `mixed` qubits per block
    (the structure tilesim::mixed_bits / split_blocks detect)."""
    targets = sorted(mixed + block)
    k = len(targets)
    rng = np.random.default_rng(seed)
    m = np.zeros((1 << k, 1 << k), complex)
    for jb in range(1 << len(block)):
        u = ob.random_unitary(len(mixed), int(rng.integers(1000)))
        idx = []
        for je in range(1 << len(mixed)):
            f = 0
            for b, q in enumerate(mixed):
                f |= ((je >> b) & 1) << targets.index(q)
            for b, q in enumerate(block):
                f |= ((jb >> b) & 1) << targets.index(q)
            idx.append(f)
        m[np.ix_(idx, idx)] = u
    return targets, m
