#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02u; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python scripts/prof_pass.py rqc 30 5 f64 > $O/steps_rqc30_jit.txt 2>&1
TSG_DMMA_JIT=0 timeout 600 python scripts/prof_pass.py rqc 30 5 f64 > $O/steps_rqc30_nojit.txt 2>&1
bash scripts/ab_bench.sh "TSG_DMMA_JIT=0" "TSG_DMMA_JIT=1" > $O/ab.txt 2>&1
echo done
