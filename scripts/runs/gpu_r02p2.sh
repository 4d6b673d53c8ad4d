#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02p2; mkdir -p $O
timeout 600 python scripts/e2e_phases.py > $O/e2e_phases.txt 2>&1
timeout 600 python scripts/prof_pass.py qaoa 30 2 f32 4 > $O/steps_qaoa30_k2.txt 2>&1
timeout 600 python scripts/prof_pass.py rqc 30 5 f64 > $O/steps_rqc30.txt 2>&1
TSG_PASS_DEBUG=1 timeout 600 python -c "
import paper_2503_19894_b200 as ts
f,_=ts.run_fusion(ts.gen_benchmark('qaoa',30,4,42),ts.FusionConfig(k_max=2)); p=ts.Program(f,'f32')" > $O/qaoa_k2_passes.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsg_pass_jit -s 3 -c 1 -o $O/full_pass_qaoa30_k2 python scripts/prof_pass.py qaoa 30 2 f32 4 > $O/ncu_q.log 2>&1
echo done
