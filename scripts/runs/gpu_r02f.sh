#!/bin/bash
mkdir -p gpurun_out
PB_FORCE=1 timeout 600 python scripts/pass_bench.py "gen ks" "perm" "empty" > gpurun_out/r02f_forced_f64.txt 2>&1
PB_FORCE=1 PB_PREC=f32 timeout 600 python scripts/pass_bench.py "gen ks" "perm" "empty" > gpurun_out/r02f_forced_f32.txt 2>&1
cat gpurun_out/r02f_forced_f64.txt gpurun_out/r02f_forced_f32.txt | cut -c1-130
