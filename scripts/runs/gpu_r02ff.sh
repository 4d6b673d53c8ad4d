#!/bin/bash
# complex64 INT8 tensor-core products: digit-extraction slicing vs the three-stage rounding
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02ff; mkdir -p $O
timeout 900 python -m pytest tests/test_umma.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "umma or f32 or 32" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
PB_ROOT=abvar/umma_old timeout 600 python scripts/umma_bench.py 30 4 5 > $O/umma_old_$i.txt 2>&1
timeout 600 python scripts/umma_bench.py 30 4 5 > $O/umma_new_$i.txt 2>&1
done
timeout 600 python scripts/umma_check.py > $O/umma_check.txt 2>&1
echo done
