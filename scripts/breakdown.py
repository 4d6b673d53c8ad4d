"""Per-step kernel breakdown of one fused circuit at n qubits (device seconds
from events around every launch).  usage: breakdown.py KIND N DEPTH PREC KMAX [SEED]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402

kind, n, depth, prec, kmax = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
seed = int(sys.argv[6]) if len(sys.argv) > 6 else (7 if kind == "qaoa" else 42)
fused, st = ts.run_fusion(ts.gen_benchmark(kind, n, depth, seed), ts.FusionConfig(k_max=kmax))
prog = ts.Program(fused, prec)
sv = ts.Statevector(n, prec).init_zero()
prog.run(sv)
secs, rep = prog.run_profiled(sv)
agg = collections.defaultdict(lambda: [0, 0, 0.0])
for s in prog.steps():
    a = agg[s["kernel"]]
    a[0] += 1
    a[1] += s["n_gates"]
    a[2] += secs[s["first_gate"]]
print(f"{kind}-{n} {prec} k<={kmax}: {st['original_gate_count']} -> {st['fused_block_count']} gates, "
      f"{len(prog.steps())} steps, {rep['execution_s'] * 1e3:.1f} ms")
for k, (cnt, g, t) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    print(f"  {k:34s} {cnt:4d} launches {g:4d} gates {t * 1e3:8.2f} ms")
