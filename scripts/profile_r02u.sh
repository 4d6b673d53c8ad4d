#!/bin/bash
# Round-2 final validation + measurement pass on the final tree (transposed
# DMMA products): GPU tests and smoke first, then the bench (both arms, the
# driver's step counts), the launch list, one ncu full capture of the dominant
# kernel class, per-step listings.  Run under gpurun from the repo root.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02u
mkdir -p $O
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt; free -g >> $O/host.txt; nvidia-smi -q | grep -iE "power limit|max clocks" -A2 >> $O/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 5 --breakdown > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
echo "ref rc=$?" >> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream_dmma|tsg_dmma_jit" -s 8 -c 1 \
    -o $O/full_dmma5_rqc30 python scripts/prof_pass.py rqc 30 5 f64 > $O/ncu_full1.log 2>&1
for c in "qft 30 5 f64" "rqc 30 5 f64" "qaoa 30 5 f32 4"; do
  timeout 600 python scripts/prof_pass.py $c > "$O/steps_$(echo $c | tr ' ' '_').txt" 2>&1
done
timeout 600 python scripts/gate_times.py rqc 30 20 f64 5 > $O/gate_times_rqc30.txt 2>&1
echo done
