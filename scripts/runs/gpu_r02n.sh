#!/bin/bash
# full GPU tier + smoke + long fuzz (shuffle layouts, ks6 DMMA) + bench with the QAOA sweep
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02n; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python scripts/fuzz.py 1000 250 > $O/fuzz.txt 2>&1; echo "rc=$?" >> $O/fuzz.txt
TSG_PASS_FORCE=1 timeout 900 python scripts/fuzz.py 2000 150 > $O/fuzz_forced.txt 2>&1; echo "rc=$?" >> $O/fuzz_forced.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
