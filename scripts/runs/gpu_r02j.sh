#!/bin/bash
# warp-shuffle layout changes in tile passes: parity, per-pass times, A/B
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pass_jit.py tests/test_pass.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in "qft 30 5 f64" "rqc 30 5 f64" "qaoa 30 5 f32 4" "hes 30 5 f32 6"; do
  f=$(echo $c | tr ' ' '_')
  timeout 600 python scripts/prof_pass.py $c > "$O/steps_$f.txt" 2>&1
  TSG_PASS_SHFL=0 timeout 600 python scripts/prof_pass.py $c > "$O/steps_${f}_noshfl.txt" 2>&1
done
bash scripts/ab_bench.sh "TSG_PASS_SHFL=0" "TSG_PASS_SHFL=1" > $O/ab.txt 2>&1
echo done
