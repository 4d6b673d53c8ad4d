#!/bin/bash
# final build with TMA tile loads: fuzz (default, write-back TMA mode 3, forced passes, sharded),
# compute-sanitizer (default and mode 3), full-size extra parity
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02fz; mkdir -p $O
timeout 1200 python scripts/fuzz.py 11000 400 > $O/fuzz.txt 2>&1; echo "rc=$?" >> $O/fuzz.txt
TSG_DMMA_TMA=3 timeout 900 python scripts/fuzz.py 12000 200 > $O/fuzz_tma3.txt 2>&1; echo "rc=$?" >> $O/fuzz_tma3.txt
TSG_PASS_FORCE=1 timeout 900 python scripts/fuzz.py 13000 200 > $O/fuzz_forced.txt 2>&1; echo "rc=$?" >> $O/fuzz_forced.txt
timeout 900 python scripts/fuzz_shard.py 14000 150 > $O/fuzz_shard.txt 2>&1; echo "rc=$?" >> $O/fuzz_shard.txt
bash scripts/gpu_sanitize.sh
TSG_DMMA_TMA=3 bash scripts/gpu_sanitize.sh
timeout 2400 python scripts/fullsize_extra.py > $O/fullsize_extra.txt 2>&1; echo "rc=$?" >> $O/fullsize_extra.txt
echo done
