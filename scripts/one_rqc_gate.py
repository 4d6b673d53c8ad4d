"""One RQC-30 fused gate (index argv[1]) applied three times as standalone launches; device ms per launch (variant A/B, ncu target)."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2503_19894_b200 as ts
f, _ = ts.run_fusion(ts.gen_benchmark("rqc", 30, 20, 42), ts.FusionConfig(k_max=5))
g = f.gate(int(sys.argv[1]))
c = ts.Circuit(30)
for _ in range(3):
    c.add_matrix(list(g.targets), np.asarray(g.matrix))
os.environ["TSG_NO_PASS"] = "1"
p = ts.Program(c, "f64")
sv = ts.Statevector(30, "f64").init_random(1)
p.run(sv, use_graph=False)
secs, _ = p.run_profiled(sv)
print(sys.argv[1], [s["kernel"] for s in p.steps()], p.jit_kernels(), [round(x * 1e3, 3) for x in secs])
