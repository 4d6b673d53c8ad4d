#!/bin/bash
# functional check of the sharded bench path (N ranks on one GPU: timings not meaningful)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02cc; mkdir -p $O
timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --no-aux > $O/bench_n2.json 2> $O/bench_n2.err; echo "rc=$?" >> $O/bench_n2.err
timeout 900 python bench.py --gpus 4 --steps 2 --warmup 1 --no-aux > $O/bench_n4.json 2> $O/bench_n4.err; echo "rc=$?" >> $O/bench_n4.err
timeout 900 python bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $O/bench_ref_n2.json 2> $O/bench_ref_n2.err; echo "rc=$?" >> $O/bench_ref_n2.err
echo done
