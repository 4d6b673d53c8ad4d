# Round-1 measurement pass, tile-pass build (run under gpurun from the repo root).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 1200 python bench.py --breakdown > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
# full captures at the bench size (n = 30): first dense ks=5 DMMA launch of RQC-30,
# the largest QFT-30 tile pass, a ks=4 DMMA launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_dmma -s 0 -c 1 \
    -o gpurun_out/full_dmma5_n30 python scripts/prof_pass.py rqc 30 5 f64 > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 2 -c 1 \
    -o gpurun_out/full_pass_qft30 python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/ncu_full2.log 2>&1
timeout 600 python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/steps_qft30.txt 2>&1
timeout 600 python scripts/prof_pass.py rqc 30 5 f64 > gpurun_out/steps_rqc30.txt 2>&1
