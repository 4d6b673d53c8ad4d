#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02bb; mkdir -p $O
for gi in 5 7 23; do
  python scripts/one_rqc_gate.py $gi >> $O/times.txt 2>&1
  TSG_DMMA_JIT=2 python scripts/one_rqc_gate.py $gi >> $O/times.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stream_dmma|tsg_dmma_jit" -s 1 -c 1 -o $O/gen_g5 python scripts/one_rqc_gate.py 5 > $O/ncu1.log 2>&1
TSG_DMMA_JIT=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stream_dmma|tsg_dmma_jit" -s 1 -c 1 -o $O/jit_g5 python scripts/one_rqc_gate.py 5 > $O/ncu2.log 2>&1
echo done
