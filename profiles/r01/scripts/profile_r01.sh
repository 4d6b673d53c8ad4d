# Round-1 measurement pass (run under gpurun from the repo root).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 1200 python bench.py --breakdown > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_dmma -s 1 -c 1 \
    -o gpurun_out/prof_dmma5 python scripts/one_gate.py 28 f64 20,21,22,23,24 > gpurun_out/ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_diag -s 1 -c 1 \
    -o gpurun_out/prof_diag python scripts/one_gate.py 28 f64 3,9,17,25 diag > gpurun_out/ncu_full2.log 2>&1
