#!/bin/bash
# sorted element order unless the reorder makes the product sparse; TMA loads (mode 1)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02pm; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python scripts/low5_probe.py > $O/low5.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 600 python scripts/gate_times.py rqc 30 20 f64 5 > $O/gate_times_rqc30.txt 2>&1
for c in "qft 30 5 f64" "rqc 30 5 f64"; do timeout 600 python scripts/prof_pass.py $c > "$O/steps_$(echo $c | tr " " "_").txt" 2>&1; done
echo done
