#!/bin/bash
# final-build fusion sweep (k = 1..6 + adaptive) and a bench run
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02s; mkdir -p $O
timeout 2400 python scripts/calibrate.py --out $O --tag _r02s > $O/calibrate.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
