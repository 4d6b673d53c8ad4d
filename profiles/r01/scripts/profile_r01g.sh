# Round-1 measurement pass (final build, r01g) (run under gpurun from the repo root).
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
    -o gpurun_out/full_dmma5_n30g python scripts/prof_pass.py rqc 30 5 f64 > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 2 -c 1 \
    -o gpurun_out/full_pass_qft30g python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/ncu_full2.log 2>&1
timeout 600 python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/steps_qft30.txt 2>&1
timeout 600 python scripts/prof_pass.py rqc 30 5 f64 > gpurun_out/steps_rqc30.txt 2>&1
# complex64 INT8 tensor-core product (QAOA-30 c64, first k_stream_umma launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_umma -s 0 -c 1 \
    -o gpurun_out/full_umma_qaoa30g python scripts/prof_pass.py qaoa 30 5 f32 4 > gpurun_out/ncu_full3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_dmma -s 0 -c 1 \
    -o gpurun_out/full_dmma4_hes30g python scripts/prof_pass.py hes 30 5 f64 > gpurun_out/ncu_full4.log 2>&1
timeout 600 python scripts/prof_pass.py qaoa 30 5 f32 4 > gpurun_out/steps_qaoa30_c64.txt 2>&1
timeout 600 python scripts/breakdown.py qaoa 30 4 f32 5 > gpurun_out/breakdown_qaoa30_c64.txt 2>&1
timeout 600 python scripts/breakdown.py hes 30 20 f32 5 > gpurun_out/breakdown_hes30_c64.txt 2>&1
timeout 600 python scripts/umma_bench.py 30 4 5 > gpurun_out/umma_bench.txt 2>&1
timeout 600 python scripts/permute_bench.py 30 f64 > gpurun_out/permute_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_stream_dmmaIdLi5ELi2ELb1E -s 2 -c 1 -o gpurun_out/full_dmma5sparse_n30g \
    python scripts/prof_pass.py rqc 30 5 f64 > gpurun_out/ncu_g5.log 2>&1
timeout 600 python scripts/fuzz.py 1000 200 16 > gpurun_out/fuzz.txt 2>&1
