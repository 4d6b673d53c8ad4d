#!/bin/bash
# dense 5-qubit RQC-30 gates: timing + one ncu full capture each (targets 0..4, 3..7, 25..29)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02d5; mkdir -p $O
for i in 8 18 46 26; do timeout 300 python scripts/one_rqc_gate.py $i >> $O/times.txt 2>&1; done
for i in 8 18 46; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dmma --launch-skip 1 -c 1 -o $O/g$i python scripts/one_rqc_gate.py $i > $O/ncu_$i.log 2>&1
done
echo done
