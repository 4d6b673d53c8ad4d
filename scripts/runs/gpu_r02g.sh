#!/bin/bash
mkdir -p gpurun_out
TSG_SKIP_FULLSIZE=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02g_pytest.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r02g_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
echo "bench rc=$?"; tail -8 gpurun_out/r02g_bench.err
python -c "import json;d=json.load(open('gpurun_out/r02g_bench.json'));print(d['value'],d['per_circuit_s'],d['aux'])"
for c in "hes 30 5 f32" "qaoa 30 5 f32"; do timeout 300 python scripts/prof_pass.py $c 20 | tail -1; done
