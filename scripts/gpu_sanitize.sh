#!/bin/bash
# compute-sanitizer memcheck / racecheck over small-state runs of the new paths
# (+ TMA tensor-map tile copies: 5-qubit products on qubits 0..4 and on
# scattered high qubits, complex64 tensor-core products; $TSG_DMMA_TMA as set)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/sanitize${TSG_DMMA_TMA:+_tma$TSG_DMMA_TMA}; mkdir -p $O
cat > /tmp/san_case.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2503_19894_b200 as ts
os.environ["TSG_PASS_JIT_MIN_N"] = "1"
for kind, n, depth, k, prec in (("qft", 14, 1, 5, "f64"), ("rqc", 14, 6, 5, "f64"), ("qaoa", 14, 2, 3, "f32"),
                                ("hes", 14, 2, 5, "f32")):
    f, _ = ts.run_fusion(ts.gen_benchmark(kind, n, depth, 3), ts.FusionConfig(k_max=k))
    p = ts.Program(f, prec)
    sv = ts.Statevector(n, prec).init_random(1)
    p.run(sv, use_graph=False)
    print(kind, p.pass_layouts(), p.jit_kernels())
# a 6-qubit complex128 DMMA product and a gather
rng = np.random.default_rng(4)
c = ts.Circuit(14)
m = rng.normal(size=(64, 64)) + 1j * rng.normal(size=(64, 64))
c.add_matrix([0, 2, 4, 6, 8, 10], m / 8)
os.environ["TSG_NO_PASS"] = "1"
p = ts.Program(c, "f64")
sv = ts.Statevector(14, "f64").init_random(2)
p.run(sv, use_graph=False)
print([s["kernel"] for s in p.steps()], sv.gather([0, 5, 16383]))
for prec, tg in (("f64", [0, 1, 2, 3, 4]), ("f64", [6, 8, 10, 12, 13]), ("f32", [9, 10, 11, 12, 13]), ("f64", [8, 9, 10, 11])):
    c = ts.Circuit(14)
    m = rng.normal(size=(1 << len(tg), 1 << len(tg))) + 1j * rng.normal(size=(1 << len(tg), 1 << len(tg)))
    c.add_matrix(tg, m / 8)
    p = ts.Program(c, prec)
    sv = ts.Statevector(14, prec).init_random(3)
    p.run(sv, use_graph=False)
    print(prec, tg, [s["kernel"] for s in p.steps()], sv.gather([1, 77]))
PY
timeout 1200 compute-sanitizer --tool memcheck --leak-check no python /tmp/san_case.py > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
timeout 1200 compute-sanitizer --tool racecheck python /tmp/san_case.py > $O/racecheck.txt 2>&1; echo "rc=$?" >> $O/racecheck.txt
echo done
