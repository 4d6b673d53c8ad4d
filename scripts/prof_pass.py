"""Profiling driver: run one fused circuit as a Program (tile passes on) so
ncu can capture k_pass launches.  usage: prof_pass.py KIND N KMAX PREC [DEPTH]"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402

kind, n, kmax, prec = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
depth = int(sys.argv[5]) if len(sys.argv) > 5 else (1 if kind == "qft" else 20)
fused, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 42), ts.FusionConfig(k_max=kmax))
prog = ts.Program(fused, prec)
sv = ts.Statevector(n, prec).init_basis(5)
prog.run(sv, use_graph=False)
secs, rep = prog.run_profiled(sv)
for st in prog.steps():
    print(f"{st['kernel']:24s} gates {st['first_gate']:4d}+{st['n_gates']:3d} high {st['high']} "
          f"{secs[st['first_gate']]*1e3:8.3f} ms")
print("total", rep["execution_s"])
