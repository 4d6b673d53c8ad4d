"""Validate bench.py's stratified CPU sample against a FULL CPU run of the
30-qubit step (fused QFT-30 + RQC-30, complex128, k <= 5) on this host.

Writes gpurun_out/cpu_full_validate.json: the sampled estimate (bench.py's
CpuStep, every fused gate over 1/S of its group range, scaled by S) next to
the measured seconds of the oracle's complete run_circuit over both circuits.
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import binding as ob  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    threads = os.cpu_count() or 1
    cs = bench.CpuStep(n, 5, threads)
    budget = 180.0 / 25
    cs.calibrate(budget)
    samples = [cs.run() for _ in range(6)]
    est = statistics.median(s[1] for s in samples)
    # full run of both circuits from the basis state
    cs.re.fill(0.0)
    cs.im.fill(0.0)
    cs.re[0x2AAAAAAA & ((1 << n) - 1)] = 1.0
    t0 = time.perf_counter()
    per = {}
    for kind, c, _ in cs.circs:
        r = ob.run_circuit(c, cs.re, cs.im, threads=threads, s=1)
        per[kind] = r["planning_s"] + r["execution_s"]
    wall = time.perf_counter() - t0
    out = {"n": n, "threads": threads, "slices": cs.slices, "sampled_estimates_s": [s[1] for s in samples],
           "sampled_estimate_median_s": est, "full_run_s": sum(per.values()), "full_run_wall_s": wall,
           "full_run_per_circuit_s": per, "ratio_estimate_over_full": est / sum(per.values()),
           "fused_stream_sha16": cs.sha16, "norm_after_full_run": ob.norm(cs.re, cs.im)}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "cpu_full_validate.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
