"""Pass planner A/B: device seconds per circuit (30 qubits) for the in-order
greedy planner (TSG_PASS_LOOKAHEAD=0) and the commutation-aware lookahead
planner (default), over fusion widths.  The planner choice is read once per
process, so each setting runs in its own process:
  python scripts/planner_ab.py [--precompile]      (spawns both settings)"""
import json
import os
import subprocess
import sys

CASES = [("qft", 1, 0, "f64"), ("rqc", 20, 42, "f64"), ("qaoa", 4, 7, "f32"), ("hes", 6, 42, "f32"),
         ("ala", 20, 42, "f64")]
KS = (1, 2, 3, 4, 5)


def child(precompile):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2503_19894_b200 as ts
    out = {}
    svs = {}
    for kind, depth, seed, prec in CASES:
        for k in KS:
            f, _ = ts.run_fusion(ts.gen_benchmark(kind, 30, depth, seed), ts.FusionConfig(k_max=k))
            if precompile:
                ts.pass_jit_precompile(f, prec)
                continue
            if prec not in svs:
                svs[prec] = ts.Statevector(30, prec).init_basis(0)
            sv = svs[prec]
            p = ts.Program(f, prec)
            p.run(sv)
            t = sorted(p.run(sv)["execution_s"] for _ in range(3))[1]
            st = p.steps()
            out[f"{kind}-k{k}"] = {"s": t, "steps": len(st), "passes": sum(s["kind"] == "pass" for s in st)}
            del p
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(len(sys.argv) > 2 and sys.argv[2] == "pre")
        sys.exit(0)
    pre = "--precompile" in sys.argv
    res = {}
    for w in ("0", "256"):
        env = dict(os.environ, TSG_PASS_LOOKAHEAD=w)
        r = subprocess.run([sys.executable, __file__, "--child", "pre" if pre else "run"], env=env,
                           capture_output=True, text=True)
        if r.returncode != 0:
            print(r.stderr[-3000:])
            sys.exit(1)
        res[w] = json.loads(r.stdout.strip().splitlines()[-1]) if not pre else {}
    if pre:
        print("precompiled")
        sys.exit(0)
    for key in res["0"]:
        a, b = res["0"][key], res["256"][key]
        print(f"{key:10s} in-order {a['s']*1e3:8.2f} ms ({a['steps']:3d} steps, {a['passes']:3d} passes)   "
              f"lookahead {b['s']*1e3:8.2f} ms ({b['steps']:3d} steps, {b['passes']:3d} passes)  {b['s']/a['s']:.3f}")
