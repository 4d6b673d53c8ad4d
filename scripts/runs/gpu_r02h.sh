#!/bin/bash
# Re-entry check: GPU tests, smoke, a short bench on a fresh box.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02h; mkdir -p $O
nvidia-smi -q | grep -iE "power limit|max clocks" -A2 > $O/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
