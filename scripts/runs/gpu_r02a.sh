#!/bin/bash
# round-2 first GPU call: full-size parity, bench (both arms), CPU-sample validation
set -x
mkdir -p gpurun_out
nproc > gpurun_out/r02a_host.txt; free -g >> gpurun_out/r02a_host.txt; lscpu | grep "Model name" >> gpurun_out/r02a_host.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r02a_fullsize.log 2>&1
echo "fullsize rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo "bench rc=$?"
timeout 400 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r02a_bench_ref.json 2> gpurun_out/r02a_bench_ref.err
echo "ref rc=$?"
timeout 900 python scripts/cpu_full_validate.py > gpurun_out/r02a_cpuval.log 2>&1
echo "cpuval rc=$?"
tail -5 gpurun_out/r02a_fullsize.log
