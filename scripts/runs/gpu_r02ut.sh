#!/bin/bash
# k_stream_umma with TMA tensor-map tile loads: parity, A/B vs bulk copies (TSG_DMMA_TMA=0)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02ut; mkdir -p $O
timeout 900 python -m pytest tests/test_umma.py tests/test_gpu_tma.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for m in 1 0 1 0; do
  echo "== tma=$m" >> $O/umma.txt
  TSG_DMMA_TMA=$m timeout 600 python scripts/umma_bench.py >> $O/umma.txt 2>&1
  echo "qaoa tma=$m $(TSG_DMMA_TMA=$m timeout 600 python scripts/prof_pass.py qaoa 30 5 f32 4 | tail -1)" >> $O/qaoa.txt
done
echo done
