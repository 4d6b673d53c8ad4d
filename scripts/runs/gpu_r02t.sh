#!/bin/bash
# JIT DMMA products (zero tiles compiled out): parity, per-gate timing, A/B
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02t; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python scripts/prof_pass.py rqc 30 5 f64 > $O/steps_rqc30_jit.txt 2>&1
TSG_DMMA_JIT=0 timeout 600 python scripts/prof_pass.py rqc 30 5 f64 > $O/steps_rqc30_nojit.txt 2>&1
bash scripts/ab_bench.sh "TSG_DMMA_JIT=0" "TSG_DMMA_JIT=1" > $O/ab.txt 2>&1
echo done
