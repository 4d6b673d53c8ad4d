import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2503_19894_b200 as ts
for n in [int(a) for a in sys.argv[1:]] or [20, 26, 28, 30]:
    for kind, depth in (("qft", 1), ("rqc", 20)):
        c = ts.gen_benchmark(kind, n, depth, 42)
        f, st = ts.run_fusion(c, ts.FusionConfig(k_max=5))
        sv = ts.Statevector(n, "f64").init_basis(0x2AAAAAAA & ((1 << n) - 1))
        prog = ts.Program(f, "f64")
        secs, rep = prog.run_profiled(sv)
        nrm = sv.norm()
        bad = None
        if abs(nrm - 1) > 1e-9:
            # bisect: rerun gate by gate checking the norm
            sv.init_basis(0x2AAAAAAA & ((1 << n) - 1))
            for i, g in enumerate(f.gates()):
                p = ts.KernelPlan(g, n)
                ts.apply_kernel(p, sv)
                x = sv.norm()
                if abs(x - 1) > 1e-9:
                    bad = (i, g.targets, p.info(), x)
                    break
        print(n, kind, st["fused_block_count"], f"norm-1={nrm-1:.3e}", f"t={rep['execution_s']*1e3:.2f}ms", bad, flush=True)
