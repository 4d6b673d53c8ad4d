"""B200 cost-model calibration and fusion sweep (north star item 2).

  python scripts/calibrate.py [--bench-n 28] [--n 30] [--out profiles/r01]

1. bench_cost_model on the device for complex128 and complex64 -> saved in
   SPEC's text format as <out>/costmodel_b200_{f64,f32}.txt.
2. Fusion sweep: for each circuit / precision, size-only fusion k = 1..6 and
   adaptive fusion (k_max = 5 and the paper-cpu preset k_max 7 / cap 4096)
   driven by the measured model; prints fused gate count, total op count,
   model-predicted seconds and measured device seconds per circuit.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_19894_b200 as ts  # noqa: E402


def model_threads(cm):
    """The threads axis value the device bench recorded (its SM count)."""
    for line in cm.serialize().splitlines():
        for tok in line.split():
            if tok.startswith("threads="):
                return int(tok.split("=")[1])
    return 1


def predicted(cm, fused, n):
    tot = 0.0
    threads = model_threads(cm)
    for g in fused.gates():
        kp = ts.KernelPlan(g, n)
        tot += cm.estimate(g.k, kp.info()["op_count"], threads, n)
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench-n", type=int, default=28)
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="profiles/r01")
    ap.add_argument("--tag", default="", help="suffix of the sweep file (fusion_sweep<tag>.json)")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    models = {}
    for prec in ("f64", "f32"):
        t0 = time.time()
        cm = ts.bench_cost_model(args.bench_n, 6, prec, args.reps, 1)
        path = os.path.join(args.out, f"costmodel_b200_{prec}.txt")
        cm.save(path)
        models[prec] = cm
        print(f"# cost model {prec}: {time.time() - t0:.1f}s -> {path}", flush=True)
        print(cm.serialize(), flush=True)

    rows = []
    n = args.n
    circuits = [("qft", 1, "f64"), ("rqc", 20, "f64"), ("qaoa", 4, "f32")]
    for kind, depth, prec in circuits:
        c = ts.gen_benchmark(kind, n, depth, 42 if kind != "qaoa" else 7)
        cm = models[prec]
        sv = ts.Statevector(n, prec).init_zero()
        configs = [(f"size-only k={k}", ts.FusionConfig(k_max=k)) for k in range(1, 7)]
        th = model_threads(cm)  # the device bench's threads axis (its SM count)
        pc = ts.FusionConfig.paper_cpu()
        pc.threads = th
        configs += [("adaptive k_max=5", ts.FusionConfig(k_max=5, mode="adaptive", threads=th)),
                    ("adaptive k_max=6", ts.FusionConfig(k_max=6, mode="adaptive", threads=th)),
                    ("paper-cpu (adaptive k7 cap4096)", pc)]
        for name, cfg in configs:
            try:
                fused, st = ts.run_fusion(c, cfg, cm)
            except ts.TilesimError as e:
                print(f"{kind} {name}: {e}")
                continue
            try:
                prog = ts.Program(fused, prec)
            except ts.TilesimError as e:
                print(f"{kind} {name}: not runnable on the device: {e}")
                continue
            prog.run(sv)
            runs = [prog.run(sv)["execution_s"] for _ in range(2)]
            pred = predicted(cm, fused, n)
            steps = prog.steps()
            row = {"circuit": f"{kind}-{n}", "precision": prec, "fusion": name, "gates": st["fused_block_count"],
                   "original": st["original_gate_count"], "total_op_count": st["total_op_count"],
                   "fusion_s": st["fusion_wall_time"], "predicted_s": pred, "measured_s": min(runs),
                   "launch_steps": len(steps), "tile_passes": sum(s["kind"] == "pass" for s in steps)}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del prog
    with open(os.path.join(args.out, f"fusion_sweep{args.tag}.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
