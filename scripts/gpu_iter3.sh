cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/debug_stream.py > gpurun_out/debug_stream.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --breakdown --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_dmma -s 1 -c 1 -o gpurun_out/dmma5b python scripts/one_gate.py 28 f64 20,21,22,23,24 > gpurun_out/ncu_dmma5.log 2>&1
