#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pass_jit.py tests/test_gpu_parity.py tests/test_pass.py -x -q -m gpu > gpurun_out/r02d_pytest.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r02d_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
echo "bench rc=$?"; tail -12 gpurun_out/r02d_bench.err
python -c "import json;d=json.load(open('gpurun_out/r02d_bench.json'));print(d['value'],d['per_circuit_s'],d['aux'])"
timeout 300 python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/r02d_qftsteps.txt 2>&1; cat gpurun_out/r02d_qftsteps.txt
