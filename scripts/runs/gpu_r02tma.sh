#!/bin/bash
# TMA tensor-map tile copies in k_stream_dmma: parity, per-gate A/B (TSG_DMMA_TMA=0), bench
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02tma; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_umma.py tests/test_gpu_shard.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 8 18 46 26 3 13; do
  echo "tma $(timeout 300 python scripts/one_rqc_gate.py $i 2>&1 | tail -1)" >> $O/times.txt
  echo "bulk $(TSG_DMMA_TMA=0 timeout 300 python scripts/one_rqc_gate.py $i 2>&1 | tail -1)" >> $O/times.txt
done
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
TSG_DMMA_TMA=0 timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_bulk.json 2> $O/bench_bulk.err
echo done
