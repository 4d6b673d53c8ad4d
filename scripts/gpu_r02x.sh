#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02x; mkdir -p $O
timeout 900 python -m pytest tests/test_permute.py tests/test_gpu_fuzz.py tests/test_gpu_shard.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python scripts/fuzz.py 5000 200 > $O/fuzz.txt 2>&1; echo "rc=$?" >> $O/fuzz.txt
timeout 600 python scripts/prof_pass.py qft 30 5 f64 > $O/steps_qft30.txt 2>&1
TSG_NO_PERMUTE_PRE=1 timeout 600 python scripts/prof_pass.py qft 30 5 f64 > $O/steps_qft30_nopre.txt 2>&1
bash scripts/ab_bench.sh "TSG_NO_PERMUTE_PRE=1" "TSG_NO_PERMUTE_PRE=" > $O/ab.txt 2>&1
echo done
