#!/bin/bash
# TSG_DMMA_TMA modes: parity under mode 3 (loads + write-backs everywhere) and default, bench per mode
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02tma2; mkdir -p $O
TSG_DMMA_TMA=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_umma.py tests/test_gpu_shard.py tests/test_gpu_fuzz.py -m gpu -x -q -p no:cacheprovider > $O/pytest_m3.log 2>&1; echo "rc=$?" >> $O/pytest_m3.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q -p no:cacheprovider > $O/pytest_m1.log 2>&1; echo "rc=$?" >> $O/pytest_m1.log
for m in 1 0 2 3 1 0; do
  TSG_DMMA_TMA=$m timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_m$m.json 2> $O/bench_m$m.err
  python -c "
import json; d=json.loads(open('$O/bench_m$m.json').readline()); k=d['kernels']
print('mode $m', round(d['value'],4), d['clocks']['sm_mhz'], d['per_circuit_s'], {n: round(v['seconds_per_step'],4) for n,v in k.items()})" >> $O/summary.txt
done
echo done
