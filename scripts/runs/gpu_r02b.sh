#!/bin/bash
# GPU suite without the full-size cases, then the sharded bench path at world 1
mkdir -p gpurun_out
TSG_SKIP_FULLSIZE=1 timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02b_pytest.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/r02b_pytest.log
timeout 300 python bench.py --sharded --steps 2 --warmup 1 --no-aux --no-cpu-baseline > gpurun_out/r02b_sharded.json 2> gpurun_out/r02b_sharded.err
echo "sharded rc=$?"; tail -3 gpurun_out/r02b_sharded.err; cut -c1-600 gpurun_out/r02b_sharded.json
