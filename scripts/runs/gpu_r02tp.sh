#!/bin/bash
# transposed DMMA products for targets on qubit 0 (TSG_DMMA_TPOSE): parity + A/B
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02tp; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tma.py tests/test_umma.py tests/test_gpu_fuzz.py tests/test_gpu_shard.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
TSG_UMMA=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/pytest_noumma.log 2>&1; echo "rc=$?" >> $O/pytest_noumma.log
for r in 1 2; do
  for v in 1 0; do
    echo "== tpose=$v" >> $O/times.txt
    TSG_DMMA_TPOSE=$v TSG_DMMA_JIT=0 timeout 600 python scripts/variant_times.py >> $O/times.txt 2>&1
    TSG_DMMA_TPOSE=$v timeout 600 python scripts/low5_probe.py >> $O/times.txt 2>&1
    TSG_DMMA_TPOSE=$v timeout 600 python scripts/gate_times.py rqc 30 20 f64 5 > $O/gt_${v}_${r}.txt 2>&1
    echo "qaoa tpose=$v $(TSG_DMMA_TPOSE=$v timeout 600 python scripts/prof_pass.py qaoa 30 5 f32 4 | tail -1)" >> $O/times.txt
  done
done
echo done
