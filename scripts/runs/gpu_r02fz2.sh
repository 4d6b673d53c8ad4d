#!/bin/bash
# final tree (transposed DMMA products for targets on qubit 0): fuzz (default,
# forced passes, transposition off as the A side), compute-sanitizer
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02fz2; mkdir -p $O
timeout 1200 python scripts/fuzz.py 21000 400 > $O/fuzz.txt 2>&1; echo "rc=$?" >> $O/fuzz.txt
TSG_PASS_FORCE=1 timeout 900 python scripts/fuzz.py 22000 150 > $O/fuzz_forced.txt 2>&1; echo "rc=$?" >> $O/fuzz_forced.txt
TSG_NO_PASS=1 timeout 900 python scripts/fuzz.py 23000 150 > $O/fuzz_nopass.txt 2>&1; echo "rc=$?" >> $O/fuzz_nopass.txt
O=gpurun_out/r02fz2 bash scripts/gpu_sanitize.sh
echo done
