#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02dd; mkdir -p $O
timeout 1500 python bench.py --gpus 8 --steps 2 --warmup 1 --no-aux > $O/bench_n8.json 2> $O/bench_n8.err; echo "rc=$?" >> $O/bench_n8.err
echo done
