#!/bin/bash
# complex128 6-qubit DMMA: parity + timing (NRB 2 default build), ks5 regression check
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "dmma6 or apply_matches" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python scripts/d6_bench.py f64 > $O/d6_f64.txt 2>&1
timeout 300 python scripts/d5_bench.py > $O/d5.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_stream_dmma -s 2 -c 1 -o $O/full_dmma6 python scripts/one_gate.py 30 f64 6,7,8,9,10,11 dense 3 > $O/ncu6.log 2>&1
echo done
