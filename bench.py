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
             result (norm and sampled amplitudes), wall clock; the second
             circuit's host front end overlaps the first one's device run
             (Program.enqueue)
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
METRIC = "30q circuit sim time (s) + per-gate HBM GB/s vs peak"
FALLBACK_HBM_GBS = 6650.0


def config_block(n, kmax, qft_gates, rqc_gates):
    """The workload, identical in both arms (the driver compares them)."""
    return {"workload": WORKLOAD, "n_qubits": n, "precision": "complex128", "fusion": f"size-only k<={kmax}",
            "qft_gates": qft_gates, "rqc_gates": rqc_gates, "input": "basis state |0x2AAAAAAA>",
            "l2": f"state {2 ** n * 16 / 2 ** 30:g} GiB >> 126 MB L2; no flush needed"}


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


def fused_stream_sha16(gate_lists):
    """sha256 over every fused gate (int32 targets, complex128 row-major matrix)
    of the step's circuits: both arms print it, so the CPU reference arm is seen
    to time the same fused gate stream as the GPU arm."""
    import hashlib

    import numpy as np

    h = hashlib.sha256()
    for gates in gate_lists:
        for t, m in gates:
            h.update(np.asarray(t, dtype=np.int32).tobytes())
            h.update(np.ascontiguousarray(m, dtype=np.complex128).tobytes())
    return h.hexdigest()[:16]


def product_stream(fused):
    return [(g.targets, g.matrix) for g in fused.gates()]


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
    (tilesim/shard.hpp), one process per GPU; exchanges are in-place
    peer-memory kernels over CUDA IPC (NVLink / NVSwitch), pipelined with the
    local gates after them where the plan allows (strong scaling)."""
    import paper_2503_19894_b200 as ts

    if world & (world - 1):
        raise SystemExit("sharding needs a power-of-two GPU count")
    g = world.bit_length() - 1
    n = args.n
    # one GPU per rank; on a box with fewer GPUs than ranks (a functional check
    # only) ranks share devices round-robin and the line says so
    n_dev = max(1, ts.device_count())
    ctx = ts.Context(local % n_dev)

    def bcast_uid():
        obj = [ts.DistState.unique_id() if rank == 0 else None]
        if world > 1:
            dist.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    (fq, sq), (fr, sr), front_s = build_circuits(ts, n, args.kmax)
    pq, pr = ts.ShardPlan(fq, g), ts.ShardPlan(fr, g)
    d = ts.DistState(n, g, rank, bcast_uid(), "f64", ctx)
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
    # compute-only timeline (the same local segments, no exchange): exposed
    # swap time = step - compute-only
    dist.barrier()
    c_step = dist.max(sum(d.run_local_only(p)["execution_s"] for p in (pq, pr)))
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
    d.close()
    # auxiliary: SURVEY §8(d) C4 (RQC-33 c128) at this GPU count, and C5
    # (TFIM-36 c64) when 8 GPUs hold it; device seconds, median of 3
    aux = {}
    if not args.no_aux:
        for name, kind, nn, depth, prec, min_world in (("rqc33_c128", "rqc", 33, 20, "f64", 1),
                                                        ("tfim36_c64", "hes", 36, 20, "f32", 8)):
            if world < min_world:
                continue
            fa, _ = ts.run_fusion(ts.gen_benchmark(kind, nn, depth, 42), ts.FusionConfig(k_max=args.kmax))
            pa = ts.ShardPlan(fa, g)
            da = ts.DistState(nn, g, rank, bcast_uid(), prec, ctx)
            da.init_basis(0)
            da.run(pa)
            reps = [da.run(pa) for _ in range(3)]
            secs = sorted(dist.max(r["execution_s"]) for r in reps)[1]
            comp = dist.max(da.run_local_only(pa)["execution_s"])
            ia = pa.info()
            aux[name] = {"seconds": secs, "compute_only_s": comp, "exposed_exchange_s": max(0.0, secs - comp),
                         "exchange_s": dist.max(statistics.median(r["exchange_s"] for r in reps)),
                         "exchanges": ia["exchanges"], "pipelined_exchanges": ia["pipelined_exchanges"],
                         "bytes_sent_per_rank": reps[0]["exchanged_bytes"]}
            da.close()
    if rank == 0:
        iq, ir = pq.info(), pr.info()
        sent = xbytes / max(1, args.steps)
        print(json.dumps({
            "metric": METRIC, "value": t_step, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated QFT-30 / RQC-30 circuits, basis-state input)",
            "config": config_block(n, args.kmax, f"{sq['original_gate_count']}->{sq['fused_block_count']}",
                                   f"{sr['original_gate_count']}->{sr['fused_block_count']}"),
            "parallelism": f"{g} global qubits over {world} GPUs (one process per GPU, peer-memory exchanges)"
                           + ("" if n_dev >= world else f"; FUNCTIONAL CHECK ONLY: {world} ranks share {n_dev} GPU(s)"),
            "fused_stream_sha16": fused_stream_sha16([product_stream(fq), product_stream(fr)]),
            "exchange": {"exchanges_per_step": iq["exchanges"] + ir["exchanges"],
                         "pipelined_per_step": iq["pipelined_exchanges"] + ir["pipelined_exchanges"],
                         "rank_blocks_per_step": iq["rank_blocks"] + ir["rank_blocks"],
                         "seconds_per_step": x_step, "bytes_sent_per_rank_per_step": int(sent),
                         "nvlink_GBps": sent / x_step / 1e9 if x_step > 0 else None,
                         "nvlink_frac_of_900": sent / x_step / 900e9 if x_step > 0 else None,
                         "compute_only_s_per_step": c_step, "exposed_s_per_step": max(0.0, t_step - c_step)},
            "front_end_s": front_s, "gpu_launches": launches, "clocks": clock_info, "e2e": e2e,
            "cpu_baseline": None, "aux": aux}))
    dist.close()


def qft20_vs_oracle(ts, ctx):
    """BASELINE configs[0]: QFT-20 on |0x5A5A5>, reference fusion
    k <= 3, GPU device seconds next to the CPU oracle's full run_circuit
    (all host threads) and the max |dpsi| between the two."""
    import numpy as np

    from oracle import binding as ob

    n1, x = 20, 0x5A5A5
    f1, st1 = ts.run_fusion(ts.gen_benchmark("qft", n1), ts.FusionConfig(k_max=3))
    p1 = ts.Program(f1, "f64", ctx=ctx)
    s1 = ts.Statevector(n1, "f64", ctx=ctx)
    secs = []
    for _ in range(5):
        s1.init_basis(x)
        secs.append(p1.run(s1)["execution_s"])
    s1.init_basis(x)
    p1.run(s1)
    o = ob.Circuit(n1)
    for g in f1.gates():
        o.add_matrix(g.targets, g.matrix)
    re = np.zeros(1 << n1)
    im = np.zeros(1 << n1)
    re[x] = 1.0
    threads = os.cpu_count() or 1
    r = ob.run_circuit(o, re, im, threads=threads, s=1)
    return {"seconds": sorted(secs)[2], "gates": f"{st1['original_gate_count']}->{st1['fused_block_count']}",
            "cpu_oracle_seconds": r["planning_s"] + r["execution_s"], "cpu_threads": threads,
            "maxdiff_vs_cpu_oracle": ts.compare_states(s1, (re, im))}


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
    # the full step's result at the 64 sampled indices: each end-to-end step
    # below must reproduce it exactly (same kernels, nothing skipped)
    pr.run(sv)
    ref_re, ref_im = sv.gather(idx[:64])

    # ---- e2e through the public API, host inputs and a host-side result
    e2e = None
    if not args.no_e2e:
        e2e_times = []
        h2d = 0
        for g in fq.gates() + fr.gates():
            h2d += g.matrix.size * 16 + 4 * len(g.targets)
        d2h = 8 + 16 * 64
        for _ in range(max(1, min(args.steps, 3))):  # median of up to 3 end-to-end steps
            # The public API pipelined: QFT-30 is generated, fused, planned,
            # uploaded and enqueued (Program.enqueue, asynchronous on the state's
            # stream); RQC-30's generation, fusion, planning and matrix upload
            # then run on the host while QFT executes; the norm reduction
            # synchronises.  Same work, same copies as a sequential step.
            t0 = time.perf_counter()
            sv.init_basis(x)  # asynchronous: the state's reset overlaps QFT-30's host front end
            cfg = ts.FusionConfig(k_max=args.kmax)
            fq2, _ = ts.run_fusion(ts.gen_benchmark("qft", n), cfg)
            p1 = ts.Program(fq2, "f64", ctx=ctx)
            p1.enqueue(sv)
            fr2, _ = ts.run_fusion(ts.gen_benchmark("rqc", n, 20, 42), cfg)
            p2 = ts.Program(fr2, "f64", ctx=ctx)
            p2.enqueue(sv)
            nrm = sv.norm()
            got_re, got_im = sv.gather(idx[:64])  # 64 sampled amplitudes: one device gather, one copy back
            e2e_times.append(time.perf_counter() - t0)
            del p1, p2
            # one_tol=1e-8 lowering of cos(phi)~1 in tiny CP phases perturbs the norm by ~1e-8 (SPEC semantics)
            assert abs(nrm - 1.0) < 1e-6, nrm
            assert np.array_equal(got_re, ref_re) and np.array_equal(got_im, ref_im), "e2e step != timed step"
        e2e = {"value": dist.max(statistics.median(e2e_times)), "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "includes": "generate+fuse+plan+upload+init+run+readback",
               "pipelining": "RQC-30's host front end (generate, fuse, plan, upload) overlaps QFT-30's device run "
                             "(Program.enqueue); the norm reduction synchronises",
               "readback": "the state's norm (device reduction) and 64 sampled amplitudes, not the 16 GiB state",
               "check": "every e2e step's 64 sampled amplitudes equal the device-timed step's bit for bit",
               "note": "wall clock with host gaps between steps: the power-capped GPU clocks higher than in the "
                       "back-to-back device-timed loop, so e2e can come out below `value`"}

    cpu = None
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        cpu = cpu_baseline(n, args.kmax, args.cpu_seconds)

    # auxiliary (not the headline), device seconds, median of 3 after warm-up:
    #   BASELINE.json configs[2]: QAOA-30 (p = 4) complex64, fusion k <= 5, and
    #                             its size-only fusion sweep k = 1..6
    #   SURVEY §8(d) C2b dense class: ALA-30 (depth 20, seed 42) complex128, k <= 5
    #   configs[0] / C1: QFT-20 complex128, fusion k <= 3, against the CPU oracle
    #                    run in full on this host (parity and CPU seconds)
    aux = None
    if not args.no_aux and world == 1:
        aux = {}

        def dev_seconds(prog, state):
            for _ in range(2):
                prog.run(state)
            return sorted(prog.run(state)["execution_s"] for _ in range(3))[1]

        qa, sqa = ts.run_fusion(ts.gen_benchmark("qaoa", n, 4, 7), ts.FusionConfig(k_max=args.kmax))
        pqa = ts.Program(qa, "f32", ctx=ctx)
        sq32 = ts.Statevector(n, "f32", ctx=ctx).init_basis(0)
        aux["qaoa30_c64_k5"] = {"seconds": dev_seconds(pqa, sq32),
                                "gates": f"{sqa['original_gate_count']}->{sqa['fused_block_count']}",
                                "steps": len(pqa.steps())}
        # configs[2]'s fusion sweep k = 1..6 (size-only) on the same circuit: the
        # tile passes take the small-k gate streams, so the best k is not the widest
        sweep = {}
        for k in range(1, 7):
            qk, sqk = ts.run_fusion(ts.gen_benchmark("qaoa", n, 4, 7), ts.FusionConfig(k_max=k))
            pk = ts.Program(qk, "f32", ctx=ctx)
            sweep[f"k={k}"] = {"seconds": dev_seconds(pk, sq32), "gates": sqk["fused_block_count"],
                               "steps": len(pk.steps())}
            del pk
        best = min(sweep, key=lambda kk: sweep[kk]["seconds"])
        aux["qaoa30_c64_sweep"] = dict(sweep, best=best)
        del pqa, sq32
        al, sal = ts.run_fusion(ts.gen_benchmark("ala", n, 20, 42), ts.FusionConfig(k_max=args.kmax))
        pal = ts.Program(al, "f64", ctx=ctx)
        sv.init_random(1)
        aux["ala30_c128_k5"] = {"seconds": dev_seconds(pal, sv),
                                "gates": f"{sal['original_gate_count']}->{sal['fused_block_count']}",
                                "steps": len(pal.steps())}
        del pal
        aux["qft20_c128_k3"] = qft20_vs_oracle(ts, ctx)
        # SURVEY §8(d) C4 at one GPU (the 1-GPU point of its 1/2/4/8 curve):
        # RQC-33 depth 20 complex128, a 128 GiB state
        f33, s33 = ts.run_fusion(ts.gen_benchmark("rqc", 33, 20, 42), ts.FusionConfig(k_max=args.kmax))
        p33 = ts.Program(f33, "f64", ctx=ctx)
        sv33 = ts.Statevector(33, "f64", ctx=ctx).init_basis(0)
        aux["rqc33_c128_k5"] = {"seconds": dev_seconds(p33, sv33),
                                "gates": f"{s33['original_gate_count']}->{s33['fused_block_count']}"}
        del p33, sv33

    out = {
        "metric": METRIC,
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
        "config": config_block(n, args.kmax, f"{sq['original_gate_count']}->{sq['fused_block_count']}",
                               f"{sr['original_gate_count']}->{sr['fused_block_count']}"),
        "parallelism": f"replicas x{world}",
        "fused_stream_sha16": fused_stream_sha16([product_stream(fq), product_stream(fr)]),
        "front_end_s": front_s,
        "per_circuit_s": {"qft30": pq.run(sv)["execution_s"], "rqc30": pr.run(sv)["execution_s"]},
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
# The reference ships no runnable simulator, so its CPU path is
# the oracle's SPEC-faithful run_circuit (specialised apply_kernel, all host
# threads; oracle/oracle.cpp).  Circuits are generated AND fused by the oracle
# itself (no product code on this leg); the fused stream's hash is printed so
# it can be matched against the GPU arm's.  A full 30-qubit step takes ~5 min
# on 16 cores, so each timed step runs EVERY fused gate over one stratum
# (1/S of its group range, a different stratum per step) and scales by S;
# profiles/r02/cpu_full_validate.json checks that estimate against a full run.
def oracle_circuits(n, kmax):
    from oracle import binding as ob

    out = []
    for kind, depth, seed in (("qft", 1, 0), ("rqc", 20, 42)):
        fused, stats = ob.run_fusion(ob.gen_benchmark(kind, n, depth, seed), mode="size", k_max=kmax)
        out.append((kind, fused, stats))
    return out


class CpuStep:
    """One bounded CPU sample of the step: every fused gate of QFT-n and RQC-n
    over stratum i of S of its group range, on a resident 2^n host state."""

    def __init__(self, n, kmax, threads):
        import numpy as np

        from oracle import binding as ob

        self.ob, self.n, self.threads = ob, n, threads
        self.circs = oracle_circuits(n, kmax)
        self.sha16 = fused_stream_sha16([[(t, m) for t, m, *_ in c.gates()] for _, c, _ in self.circs])
        self.gates_total = sum(len(c) for _, c, _ in self.circs)
        self.re = np.zeros(1 << n)
        self.im = np.zeros(1 << n)
        self.re.fill(0.0)  # first-touch the pages outside the timed region
        self.im.fill(0.0)
        self.re[0x2AAAAAAA & ((1 << n) - 1)] = 1.0
        self.slices = 1
        self.next = 0

    def run(self):
        """Returns (seconds measured, seconds scaled to the whole step, gates timed)."""
        t = 0.0
        gates = 0
        for _, c, _ in self.circs:
            r = self.ob.run_circuit_slice(c, self.re, self.im, self.next, self.slices, threads=self.threads, s=1)
            t += r["planning_s"] + r["execution_s"]
            gates += len(c)
        self.next += 1
        return t, t * self.slices, gates

    def calibrate(self, step_budget_s):
        """Pick S (a power of two) so one sampled step takes about step_budget_s."""
        self.slices = 1024
        t, full, _ = self.run()
        s = 1
        while s < 4096 and full / s > step_budget_s:
            s *= 2
        self.slices = s
        self.next = 0
        return full

    def describe(self, budget_s):
        return (f"oracle run_circuit (SPEC apply_kernel, s=1, {self.threads} threads), circuits generated and fused "
                f"by the oracle; per step every one of the {self.gates_total} fused gates over 1/{self.slices} of "
                f"its group range (a different stratum each step), scaled x{self.slices}; step budget "
                f"{budget_s:.1f}s")


def cpu_baseline(n, kmax, budget_s, samples=2):
    threads = os.cpu_count() or 1
    if _host_mem_gb() < 2.5 * (2 ** n * 16) / 1e9:
        return {"value": None, "unit": "s", "cores": threads, "kind": "port",
                "sample": f"skipped: host RAM below 2.5x the 2^{n} complex128 state"}
    cs = CpuStep(n, kmax, threads)
    cs.calibrate(budget_s / samples)
    vals = [cs.run() for _ in range(samples)]
    return {"value": statistics.median(v[1] for v in vals), "unit": "s", "cores": threads, "kind": "port",
            "sample": cs.describe(budget_s / samples), "fused_stream_sha16": cs.sha16,
            "detail": {"gates_timed": vals[-1][2], "gates_total": cs.gates_total,
                       "sample_fraction_per_step": 1.0 / cs.slices, "steps": samples,
                       "seconds_measured": [v[0] for v in vals]}}


def _host_mem_gb():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable"):
                    return int(line.split()[1]) / 1e6
    except Exception:
        pass
    return 0.0


def run_reference(args):
    """--impl reference: the CPU path (oracle port of SPEC's run_circuit) on all
    host cores, same metric/config as our arm; rank 0 only under torchrun."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n = args.n
    threads = os.cpu_count() or 1
    cs = CpuStep(n, args.kmax, threads)
    # the whole --steps K --warmup W run in about 3 minutes
    budget = max(2.0, min(args.cpu_seconds, 180.0 / max(1, args.steps + args.warmup)))
    cs.calibrate(budget)
    for _ in range(args.warmup):
        cs.run()
    vals = [cs.run() for _ in range(args.steps)]
    v = statistics.median(x[1] for x in vals)
    stats = {kind: f"{st['original_gate_count']}->{st['fused_block_count']}" for kind, _, st in cs.circs}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v,
        "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated QFT-30 / RQC-30 circuits, basis-state input)",
        "config": config_block(n, args.kmax, stats["qft"], stats["rqc"]),
        "fused_stream_sha16": cs.sha16,
        "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": "port", "sample": cs.describe(budget),
                         "detail": {"gates_timed": vals[-1][2], "gates_total": cs.gates_total,
                                    "sample_fraction_per_step": 1.0 / cs.slices,
                                    "seconds_measured_median": statistics.median(x[0] for x in vals)}},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def relaunch_under_torchrun(args):
    """--gpus N without a torchrun environment: spawn the N ranks ourselves
    (one process per GPU, rendezvous on 127.0.0.1) and pass through rank 0's
    output; returns the exit code."""
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", 0))
    if world == 0 and args.gpus > 1:
        raise SystemExit(relaunch_under_torchrun(args))
    if world and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one process per GPU")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
