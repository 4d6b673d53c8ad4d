#!/bin/bash
# ks=5 complex128: direct-out vs in-place write-back (variant inplace5), TMA modes
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02ip; mkdir -p $O
export TSG_DMMA_JIT=0
for v in base inplace5 base inplace5; do
  for m in 1 0; do
    if [ $v = base ]; then R=""; else R=paper_variants/$v; fi
    echo "== $v tma=$m" >> $O/times.txt
    PB_ROOT=$R TSG_DMMA_TMA=$m timeout 600 python scripts/variant_times.py >> $O/times.txt 2>&1
  done
done
echo done
