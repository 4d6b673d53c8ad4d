#!/bin/bash
# final round-2 measurement pass + extended parity evidence
cd ${GRAFT_REPO_ROOT:-.}
bash scripts/profile_r02v.sh > /dev/null 2>&1
O=gpurun_out/r02v
timeout 1200 python scripts/fuzz.py 7000 400 > $O/fuzz_final.txt 2>&1; echo "rc=$?" >> $O/fuzz_final.txt
TSG_PASS_FORCE=1 timeout 900 python scripts/fuzz.py 8000 200 > $O/fuzz_final_forced.txt 2>&1; echo "rc=$?" >> $O/fuzz_final_forced.txt
timeout 900 python scripts/fuzz_shard.py 9000 150 > $O/fuzz_shard_final.txt 2>&1; echo "rc=$?" >> $O/fuzz_shard_final.txt
echo done
