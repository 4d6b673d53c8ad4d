#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02aa; mkdir -p $O
timeout 1200 python -m pytest tests/test_permute.py tests/test_gpu_pass_jit.py tests/test_gpu_fuzz.py tests/test_gpu_shard.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python scripts/prof_pass.py qft 30 5 f64 > $O/steps_qft30.txt 2>&1
TSG_NO_PERM_FACTOR=1 timeout 600 python scripts/prof_pass.py qft 30 5 f64 > $O/steps_qft30_nofactor.txt 2>&1
bash scripts/ab_bench.sh "TSG_NO_PERM_FACTOR=1" "TSG_NO_PERM_FACTOR=0" > $O/ab.txt 2>&1
echo done
