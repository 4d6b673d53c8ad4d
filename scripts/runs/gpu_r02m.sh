#!/bin/bash
# fusion sweep (k = 1..6 + adaptive) with the ks6 DMMA + shuffle build; ncu of QFT-30 passes
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02m; mkdir -p $O
timeout 2400 python scripts/calibrate.py --out $O --tag _r02 > $O/calibrate.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsg_pass_jit -s 1 -c 1 \
    -o $O/full_passjit_qft30_p2 python scripts/prof_pass.py qft 30 5 f64 > $O/ncu_p2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tsg_pass_jit -s 4 -c 1 \
    -o $O/full_passjit_qft30_p5 python scripts/prof_pass.py qft 30 5 f64 > $O/ncu_p5.log 2>&1
echo done
