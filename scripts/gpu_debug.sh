cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/debug_norm.py 20 24 26 28 29 30 > gpurun_out/debug_norm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
