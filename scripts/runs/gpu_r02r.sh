#!/bin/bash
# lookahead pass planner: parity (GPU tests, fuzz) and A/B timing; bench
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02r; mkdir -p $O
timeout 1200 python -m pytest tests/test_pass.py tests/test_gpu_pass_jit.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_permute.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python scripts/fuzz.py 3000 200 > $O/fuzz.txt 2>&1; echo "rc=$?" >> $O/fuzz.txt
TSG_PASS_FORCE=1 timeout 900 python scripts/fuzz.py 4000 100 > $O/fuzz_forced.txt 2>&1; echo "rc=$?" >> $O/fuzz_forced.txt
timeout 1800 python scripts/planner_ab.py > $O/planner_ab.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
