#!/usr/bin/env python
"""bench.py -- BASELINE.json metric: 30q circuit simulation time on B200.

Workload (BASELINE.json configs[1]): QFT-30 and RQC-30 (depth 20, seed 42),
complex128, size-only fusion k <= 5, 1 B200.  One step = both fused circuits
applied back to back to a resident 2^30 statevector (16 GiB, >> the 126 MB
L2, so no L2 flush is needed between steps).

  value      device seconds per step (CUDA events on the library's stream,
             max over ranks), lower is better
  e2e        the same step through the public C ABI from host inputs:
             generate + fuse + plan/upload + init + run + read back the
             result (norm and sampled amplitudes), wall clock
  roofline   dominant kernel class: algorithmic bytes (2 * 2^n * 16 B per
             launch) / its summed per-launch event time, vs MEASURED_PEAKS.json
  cpu_baseline  the CPU oracle (SPEC-faithful run_circuit, all host cores) on
             a bounded sample of the same circuits, extrapolated per step

--impl reference times that CPU path alone (the reference ships no runnable
simulator).  N > 1 (torchrun, one process per GPU): the
same 30-qubit step sharded by log2(N) global qubits with NCCL swaps
(tilesim/shard.hpp) -- strong scaling, max over ranks.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_QUBITS = 30
WORKLOAD = "qft30+rqc30_d20_c128_sizeonly_k5"
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=N_QUBITS)
    ap.add_argument("--kmax", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-aux", action="store_true", help="skip the auxiliary QAOA-30 complex64 measurement")
    ap.add_argument("--breakdown", action="store_true", help="print the per-kernel-class table to stderr")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded (NCCL) step even on one GPU (0 global qubits: exercises that path)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Dist:
    """gloo plumbing for barrier / max-over-ranks (no data-path collective: replicas)."""

    def __init__(self, world):
        self.world = world
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        return self._reduce(x, "MAX")

    def sum(self, x: float) -> float:
        return self._reduce(x, "SUM")

    def _reduce(self, x: float, op: str) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=getattr(self.dist.ReduceOp, op))
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        reasons = set()
        for r in rows:
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def fp64_peak_tflops(clock_info):
    mhz = (clock_info or {}).get("sm_mhz") or 1965.0
    return 63.6 * 148 * 2 * mhz * 1e6 / 1e12


def build_circuits(ts, n, kmax):
    t0 = time.perf_counter()
    qft = ts.gen_benchmark("qft", n)
    rqc = ts.gen_benchmark("rqc", n, 20, 42)
    cfg = ts.FusionConfig(k_max=kmax)
    fq, sq = ts.run_fusion(qft, cfg)
    fr, sr = ts.run_fusion(rqc, cfg)
    return (fq, sq), (fr, sr), time.perf_counter() - t0


def breakdown(ts, progs, sv, n):
    """Per-kernel device time from CUDA events around every launch step
    (Program.steps(): single gates, diagonal batches and tile passes)."""
    amp = 16
    groups = {}
    for prog in progs:
        secs, _ = prog.run_profiled(sv)
        for st in prog.steps():
            s = float(secs[st["first_gate"]])  # a step's gates after its first one have zero-length marks
            info = prog.gate_info(st["first_gate"])
            key = st["kernel"]
            g = groups.setdefault(key, {"seconds": 0.0, "launches": 0, "bytes": 0, "touched": 0, "gates": 0,
                                        "flops": 0})
            g["seconds"] += s
            g["launches"] += 1
            g["gates"] += st["n_gates"]
            # algorithmic flops: 2 * op_count * 2^(n-k) per gate of the step
            gi = st["first_gate"]
            done = 0
            while done < st["n_gates"]:
                ginfo = prog.gate_info(gi)
                gi += 1
                if ginfo["kernel"] == "identity":
                    continue
                g["flops"] += 2 * ginfo["op_count"] * ginfo["loop_count"]
                done += 1
            g["bytes"] += 2 * (1 << n) * amp
            frac = info["touched_fraction"] if st["kind"] == "gate" else 1.0
            g["touched"] += int(2 * (1 << n) * amp * frac)
    return groups


def run_sharded(args, rank, world, local, dist):
    """N > 1: the same 30-qubit step sharded over N GPUs by global qubits
    (tilesim/shard.hpp), NCCL swaps, one process per GPU (strong scaling)."""
    import numpy as np  # noqa: F401

    import paper_2503_19894_b200 as ts

    if world & (world - 1):
        raise SystemExit("sharding needs a power-of-two GPU count")
    g = world.bit_length() - 1
    n = args.n
    ctx = ts.Context(local)
    if rank == 0:
        uid = ts.DistState.unique_id()
    else:
        uid = None
    if world > 1:
        import torch.distributed as tdist
        obj = [uid]
        tdist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    (fq, sq), (fr, sr), front_s = build_circuits(ts, n, args.kmax)
    pq, pr = ts.ShardPlan(fq, g), ts.ShardPlan(fr, g)
    d = ts.DistState(n, g, rank, uid, "f64", ctx)
    d.init_basis(0x2AAAAAAA & ((1 << n) - 1))
    for _ in range(args.warmup):
        d.run(pq)
        d.run(pr)
    clocks = ClockSampler(local)
    dist.barrier()
    clocks.start()
    t_dev, xs, xbytes, launches = 0.0, 0.0, 0, 0
    for _ in range(args.steps):
        for plan in (pq, pr):
            rep = d.run(plan)
            t_dev += rep["execution_s"]
            xs += rep["exchange_s"]
            xbytes += rep["exchanged_bytes"]
            launches += rep["launches"]
    clock_info = clocks.stop()
    dist.barrier()
    t_step = dist.max(t_dev / args.steps)
    x_step = dist.max(xs / args.steps)
    # e2e through the public API: generate + fuse + shard plans + init + run +
    # a host-side result (this rank's squared norm, summed over ranks)
    e2e = None
    if not args.no_e2e:
        times = []
        for _ in range(max(1, min(args.steps, 3))):  # median of up to 3 end-to-end steps
            dist.barrier()
            t0 = time.perf_counter()
            (fq2, _), (fr2, _), _ = build_circuits(ts, n, args.kmax)
            p1, p2 = ts.ShardPlan(fq2, g), ts.ShardPlan(fr2, g)
            d.init_basis(0x2AAAAAAA & ((1 << n) - 1))
            d.run(p1)
            d.run(p2)
            nrm = dist.sum(d.local_sumsq())
            times.append(time.perf_counter() - t0)
            assert abs(nrm - 1.0) < 1e-6, nrm
        h2d = sum(gt.matrix.size * 16 + 4 * len(gt.targets) for gt in fq.gates() + fr.gates())
        e2e = {"value": dist.max(statistics.median(times)), "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 8, "includes": "generate+fuse+shard-plan+init+run+norm readback"}
    if rank == 0:
        iq, ir = pq.info(), pr.info()
        print(json.dumps({
            "metric": "30q circuit sim time (s) + per-gate HBM GB/s vs peak", "value": t_step, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated QFT-30 / RQC-30 circuits, basis-state input)",
            "config": {"workload": WORKLOAD, "n_qubits": n, "precision": "complex128",
                       "fusion": f"size-only k<={args.kmax}", "parallelism": f"{g} global qubits over {world} GPUs",
                       "swaps_per_step": iq["swaps"] + ir["swaps"],
                       "rank_blocks_per_step": iq["rank_blocks"] + ir["rank_blocks"], "front_end_s": front_s},
            "exchange": {"seconds_per_step": x_step, "bytes_per_rank_per_step": xbytes // max(1, args.steps),
                         "nvlink_GBps": (xbytes / max(1, args.steps)) / x_step / 1e9 if x_step > 0 else None,
                         "exposed": "exchanges are not overlapped yet (exposed = seconds_per_step)"},
            "gpu_launches": launches, "clocks": clock_info, "e2e": e2e, "cpu_baseline": None}))
    dist.close()


def run_ours(args):
    rank, world, local = dist_env()
    dist = Dist(world)
    if world > 1 or args.sharded:
        return run_sharded(args, rank, world, local, dist)
    import numpy as np

    import paper_2503_19894_b200 as ts

    n = args.n
    ctx = ts.Context(local if world > 1 else 0)
    (fq, sq), (fr, sr), front_s = build_circuits(ts, n, args.kmax)
    pq = ts.Program(fq, "f64", ctx=ctx)
    pr = ts.Program(fr, "f64", ctx=ctx)
    sv = ts.Statevector(n, "f64", ctx)
    sv.init_basis(0x2AAAAAAA & ((1 << n) - 1))

    def step():
        pq.enqueue(sv, use_graph=True)
        pr.enqueue(sv, use_graph=True)

    for _ in range(args.warmup):
        step()
    sv.synchronize()

    clocks = ClockSampler(local)
    dist.barrier()
    sv.synchronize()
    clocks.start()
    sv.timer_begin()
    for _ in range(args.steps):
        step()
    dev_s = sv.timer_end()  # synchronizes the stream
    clock_info = clocks.stop()
    dist.barrier()
    t_step = dist.max(dev_s / args.steps)

    launches_per_step = pq.run(sv)["launches"] + pr.run(sv)["launches"]

    # ---- per-kernel breakdown + roofline (outside the timed region)
    groups = breakdown(ts, [pq, pr], sv, n)
    dom_name, dom = max(groups.items(), key=lambda kv: kv[1]["seconds"])
    peak, peak_kind = measured_peaks()
    achieved = dom["bytes"] / dom["seconds"] / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(dom_name)
        except Exception:
            traffic = None

    # ---- parity on the headline config: QFT-30 on |x> vs the closed form
    x = 0x2AAAAAAA & ((1 << n) - 1)
    sv.init_basis(x)
    pq.run(sv)
    rng = np.random.default_rng(0)
    idx = np.unique(rng.integers(0, 1 << n, 4096))
    maxdiff = 0.0
    for i0 in idx[:64]:
        re, im = sv.download(int(i0), 1)
        want = np.exp(2j * np.pi * ((x * int(i0)) % (1 << n)) / (1 << n)) / 2 ** (n / 2)
        maxdiff = max(maxdiff, abs(complex(re[0], im[0]) - want))
    qft_norm = sv.norm()

    # ---- e2e through the public API, host inputs and a host-side result
    e2e = None
    if not args.no_e2e:
        e2e_times = []
        h2d = 0
        for g in fq.gates() + fr.gates():
            h2d += g.matrix.size * 16 + 4 * len(g.targets)
        d2h = 8 + 16 * 64
        for _ in range(max(1, min(args.steps, 3))):  # median of up to 3 end-to-end steps
            t0 = time.perf_counter()
            (fq2, _), (fr2, _), _ = build_circuits(ts, n, args.kmax)
            p1 = ts.Program(fq2, "f64", ctx=ctx)
            p2 = ts.Program(fr2, "f64", ctx=ctx)
            sv.init_basis(x)
            p1.run(sv)
            p2.run(sv)
            nrm = sv.norm()
            for i0 in idx[:64]:
                sv.download(int(i0), 1)
            e2e_times.append(time.perf_counter() - t0)
            del p1, p2
            # one_tol=1e-8 lowering of cos(phi)~1 in tiny CP phases perturbs the norm by ~1e-8 (SPEC semantics)
            assert abs(nrm - 1.0) < 1e-6, nrm
        e2e = {"value": dist.max(statistics.median(e2e_times)), "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "includes": "generate+fuse+plan+upload+init+run+readback"}

    cpu = None
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        cpu = cpu_baseline(fq, fr, n, args.cpu_seconds)

    # auxiliary (not the headline): BASELINE.json config 3, QAOA-30 (p = 4)
    # complex64 with fusion k <= 5, device seconds (median of 3 after warm-up)
    aux = None
    if not args.no_aux and world == 1:
        qa, sqa = ts.run_fusion(ts.gen_benchmark("qaoa", n, 4, 7), ts.FusionConfig(k_max=args.kmax))
        pqa = ts.Program(qa, "f32", ctx=ctx)
        sq32 = ts.Statevector(n, "f32", ctx=ctx).init_basis(0)
        for _ in range(2):
            pqa.run(sq32)
        ts_q = sorted(pqa.run(sq32)["execution_s"] for _ in range(3))
        aux = {"qaoa30_c64_k5": {"seconds": ts_q[1], "gates": f"{sqa['original_gate_count']}->{sqa['fused_block_count']}",
                                 "steps": len(pqa.steps())}}
        del pqa, sq32

    out = {
        "metric": "30q circuit sim time (s) + per-gate HBM GB/s vs peak",
        "value": t_step,
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (generated QFT-30 / RQC-30 circuits, basis-state input)",
        "config": {"workload": WORKLOAD, "n_qubits": n, "precision": "complex128", "fusion": f"size-only k<={args.kmax}",
                   "qft_gates": f"{sq['original_gate_count']}->{sq['fused_block_count']}",
                   "rqc_gates": f"{sr['original_gate_count']}->{sr['fused_block_count']}",
                   "l2": "state 16 GiB >> 126 MB L2; no flush needed", "parallelism": f"replicas x{world}",
                   "front_end_s": front_s, "per_circuit_s": {"qft30": pq.run(sv)["execution_s"],
                                                             "rqc30": pr.run(sv)["execution_s"]}},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": dom_name, "peak_source": peak_kind,
                     "per_launch_bytes": 2 * (1 << n) * 16,
                     # the same kernel against the FP64 tensor (DMMA) roof: SPEC op_count flops
                     # (2 * op_count * 2^(n-k) per gate) / time vs the measured DMMA peak
                     # (63.6 MAC/clk/SM, profiles/r01/microbench.log) at the run's SM clock
                     "fp64": {"achieved_tflops": dom["flops"] / dom["seconds"] / 1e12,
                              "peak_tflops": fp64_peak_tflops(clock_info),
                              "frac": dom["flops"] / dom["seconds"] / 1e12 / fp64_peak_tflops(clock_info),
                              "peak_source": "measured DMMA.8x8x4 rate x 148 SMs x sampled SM clock"}},
        "kernels": {k: {"seconds_per_step": v["seconds"], "launches": v["launches"], "gates": v["gates"],
                        "GBps_algorithmic": v["bytes"] / v["seconds"] / 1e9,
                        "TFLOPs_algorithmic": v["flops"] / v["seconds"] / 1e12,
                        "GBps_touched": v["touched"] / v["seconds"] / 1e9} for k, v in groups.items()},
        "parity": {"qft30_analytic_maxdiff_64_samples": maxdiff, "qft30_norm": qft_norm},
        "clocks": clock_info,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "aux": aux,
    }
    if args.breakdown and rank == 0:
        for k, v in sorted(groups.items(), key=lambda kv: -kv[1]["seconds"]):
            print(f"{k:28s} {v['seconds']*1e3:9.2f} ms {v['launches']:4d} launches {v['gates']:4d} gates "
                  f"{v['bytes']/v['seconds']/1e9:8.0f} GB/s alg {v['touched']/v['seconds']/1e9:8.0f} GB/s touched",
                  file=sys.stderr)
    if rank == 0:
        print(json.dumps(out))
    dist.close()


# ----------------------------------------------------------- CPU oracle leg
def _cpu_sample(circuits, n, budget_s, threads):
    """Time the oracle's run_circuit (SPEC apply_kernel, all threads) gate by
    gate on a 2^n host state until the budget is spent; extrapolate per step."""
    import numpy as np

    from oracle import binding as ob

    re = np.zeros(1 << n)
    im = np.zeros(1 << n)
    re[0] = 1.0
    total = 0.0
    detail = []
    per_circ_budget = budget_s / len(circuits)
    for fused in circuits:
        o = ob.Circuit(n)
        for g in fused.gates():
            o.add_matrix(g.targets, g.matrix)
        G = len(o)
        spent, done = 0.0, 0
        while done < G and spent < per_circ_budget:
            t = ob.run_circuit(o, re, im, threads=threads, s=1, g_begin=done, g_end=done + 1)
            spent += t["planning_s"] + t["execution_s"]
            done += 1
        est = spent / done * G
        total += est
        detail.append({"gates_timed": done, "gates_total": G, "seconds_timed": spent, "seconds_est": est})
    return total, detail


def _host_mem_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable"):
                    return int(line.split()[1]) / 1e6
    except Exception:
        pass
    return 0.0


def cpu_baseline(fq, fr, n, budget_s):
    threads = os.cpu_count() or 1
    n_cpu = n
    scale = 1.0
    if _host_mem_gb() < 2.5 * (2 ** n * 16) / 1e9:
        n_cpu = n - 2
        scale = 4.0
    if n_cpu != n:
        import paper_2503_19894_b200 as ts
        (fq, _), (fr, _), _ = build_circuits(ts, n_cpu, 5)
    est, detail = _cpu_sample([fq, fr], n_cpu, budget_s, threads)
    return {"value": est * scale, "unit": "s", "cores": threads, "kind": "port",
            "sample": f"oracle run_circuit (SPEC apply_kernel, s=1, {threads} threads) on the first gates of the "
                      f"fused QFT/RQC circuits at n={n_cpu} within {budget_s:.0f}s, extrapolated linearly in gate "
                      f"count" + (" and x4 to n=30" if scale != 1.0 else ""),
            "detail": detail}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_2503_19894_b200 as ts  # host-only circuit generation + fusion (no GPU use)

    n = args.n
    (fq, _), (fr, _), _ = build_circuits(ts, n, args.kmax)
    budget = max(4.0, min(args.cpu_seconds, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        _cpu_sample([fq, fr], n, budget / 2, os.cpu_count() or 1)
    vals = []
    detail = None
    for _ in range(args.steps):
        v, detail = _cpu_sample([fq, fr], n, budget, os.cpu_count() or 1)
        vals.append(v)
    v = statistics.median(vals)
    threads = os.cpu_count() or 1
    print(json.dumps({
        "impl": "reference", "metric": "30q circuit sim time (s) + per-gate HBM GB/s vs peak", "value": v,
        "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated QFT-30 / RQC-30 circuits)",
        "config": {"workload": WORKLOAD, "n_qubits": n, "precision": "complex128", "fusion": f"size-only k<={args.kmax}"},
        "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": "port",
                         "sample": f"per step: oracle run_circuit on the first gates of each fused circuit within "
                                   f"{budget:.1f}s, extrapolated linearly in gate count", "detail": detail},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
