#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pass_jit.py -x -q > gpurun_out/r02e_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02e_pytest.log
timeout 600 python scripts/pass_bench.py > gpurun_out/r02e_pass_bench_f64.txt 2>&1
PB_PREC=f32 timeout 600 python scripts/pass_bench.py > gpurun_out/r02e_pass_bench_f32.txt 2>&1
cat gpurun_out/r02e_pass_bench_f64.txt gpurun_out/r02e_pass_bench_f32.txt
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:tsg_pass_jit --launch-skip 4 --launch-count 1 -f -o gpurun_out/r02e_qftpass5_jit \
  python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/r02e_ncu.log 2>&1
echo "ncu rc=$?"
