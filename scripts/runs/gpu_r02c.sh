#!/bin/bash
# ncu full captures: dense 5-qubit complex128 DMMA launch, 5th QFT-30 pass
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 $NCU --kernel-name regex:k_stream_dmma --launch-skip 1 --launch-count 1 -f -o gpurun_out/r02c_dmma5dense \
  python scripts/one_gate.py 30 f64 3,9,14,20,27 dense 2 > gpurun_out/r02c_dmma.log 2>&1
echo "dmma rc=$?"
timeout 900 $NCU --kernel-name regex:k_pass --launch-skip 4 --launch-count 1 -f -o gpurun_out/r02c_qftpass5 \
  python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/r02c_pass.log 2>&1
echo "pass rc=$?"
tail -3 gpurun_out/r02c_dmma.log gpurun_out/r02c_pass.log
