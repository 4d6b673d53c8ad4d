# Extra captures: first 5-qubit DMMA launch of RQC-30 (mangled-name match), the
# slowest QFT-30 tile pass (5th), one k_stream_umma<ks=4> launch (HES-30 c64)
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_stream_dmmaIdLi5E -s 0 -c 1 -o gpurun_out/full_dmma5k_n30 \
    python scripts/prof_pass.py rqc 30 5 f64 > gpurun_out/ncu_x1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 4 -c 1 \
    -o gpurun_out/full_pass5_qft30 python scripts/prof_pass.py qft 30 5 f64 > gpurun_out/ncu_x2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_umma -s 0 -c 1 \
    -o gpurun_out/full_umma4_hes30 python scripts/prof_pass.py hes 30 5 f32 > gpurun_out/ncu_x3.log 2>&1
