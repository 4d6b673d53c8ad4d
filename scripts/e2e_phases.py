"""Wall-clock phases of bench.py's end-to-end step (QFT-30 + RQC-30 c128)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402

n = 30
sv = ts.Statevector(n, "f64").init_zero()
for it in range(3):
    t = [time.perf_counter()]
    fq, _ = ts.run_fusion(ts.gen_benchmark("qft", n), ts.FusionConfig(k_max=5))
    fr, _ = ts.run_fusion(ts.gen_benchmark("rqc", n, 20, 42), ts.FusionConfig(k_max=5))
    t.append(time.perf_counter())
    p1 = ts.Program(fq, "f64")
    t.append(time.perf_counter())
    p2 = ts.Program(fr, "f64")
    t.append(time.perf_counter())
    sv.init_basis(5)
    r1 = p1.run(sv)
    t.append(time.perf_counter())
    r2 = p2.run(sv)
    t.append(time.perf_counter())
    sv.norm()
    t.append(time.perf_counter())
    names = ["fuse", "plan qft", "plan rqc", "run qft", "run rqc", "norm"]
    print(" ".join(f"{a}={1e3 * (t[i + 1] - t[i]):.1f}ms" for i, a in enumerate(names)),
          f"total={1e3 * (t[-1] - t[0]):.1f}ms dev={1e3 * (r1['execution_s'] + r2['execution_s']):.1f}ms")
