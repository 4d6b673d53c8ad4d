cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TSG_DMMA_MODE=direct timeout 300 python scripts/debug_stream.py > gpurun_out/debug_direct.log 2>&1
TSG_DMMA_MODE=direct timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
TSG_DMMA_MODE=direct timeout 900 python bench.py --breakdown --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
