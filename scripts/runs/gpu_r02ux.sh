#!/bin/bash
# final tree: a second driver-equivalent bench sample, and the sharded bench
# path with 2 and 4 ranks sharing this one GPU (functional check only)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02ux; mkdir -p $O
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-aux > $O/bench_n2.json 2> $O/bench_n2.err; echo "rc=$?" >> $O/bench_n2.err
timeout 900 python bench.py --gpus 4 --steps 3 --warmup 3 --no-aux > $O/bench_n4.json 2> $O/bench_n4.err; echo "rc=$?" >> $O/bench_n4.err
echo done
