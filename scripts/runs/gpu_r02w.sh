#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02w; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gather or norm" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-aux > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
