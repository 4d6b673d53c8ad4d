"""Debug helper: one synthetic block-structured gate, forced into a tile pass,
against the same gate without passes.  usage: debug_gate.py PREC N MIXED BLOCK"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402
from tests._util import random_gate_matrix  # noqa: E402

prec, n = sys.argv[1], int(sys.argv[2])
mixed = [int(x) for x in sys.argv[3].split(",")]
block = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 and sys.argv[4] else []
targets = sorted(mixed + block)
k = len(targets)
rng = np.random.default_rng(5)
m = np.zeros((1 << k, 1 << k), complex)
for jb in range(1 << len(block)):
    u = random_gate_matrix(len(mixed), int(rng.integers(1000)), "dense")
    idx = []
    for je in range(1 << len(mixed)):
        f = 0
        for b, q in enumerate(mixed):
            f |= ((je >> b) & 1) << targets.index(q)
        for b, q in enumerate(block):
            f |= ((jb >> b) & 1) << targets.index(q)
        idx.append(f)
    m[np.ix_(idx, idx)] = u
c = ts.Circuit(n)
c.add_matrix(targets, m)
c.add_matrix([0], np.diag([1, np.exp(0.3j)]))
re0 = rng.standard_normal(1 << n)
im0 = rng.standard_normal(1 << n)
out = []
for env in ({"TSG_PASS_FORCE": "1", "TSG_PASS_DEBUG": "1"}, {"TSG_NO_PASS": "1"}):
    os.environ.update(env)
    prog = ts.Program(c, prec)
    for key in env:
        os.environ.pop(key)
    sv = ts.Statevector(n, prec).upload(re0, im0)
    prog.run(sv)
    out.append(sv)
    print([s["kernel"] for s in prog.steps()])
print("diff", ts.compare_states(out[0], out[1]))
