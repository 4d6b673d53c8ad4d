#!/bin/bash
# end-to-end phases (host overheads) with the current build; ncu of dense ks5 DMMA at low / high targets
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02o; mkdir -p $O
timeout 600 python scripts/e2e_phases.py > $O/e2e_phases.txt 2>&1
TSG_PASS_SHFL=0 timeout 600 python scripts/e2e_phases.py > $O/e2e_phases_noshfl.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_dmma -s 2 -c 1 -o $O/full_dmma5_low python scripts/one_gate.py 30 f64 0,1,2,3,4 dense 3 > $O/ncu_low.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_dmma -s 2 -c 1 -o $O/full_dmma5_mid python scripts/one_gate.py 30 f64 9,10,11,12,13 dense 3 > $O/ncu_mid.log 2>&1
echo done
