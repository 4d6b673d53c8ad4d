#!/bin/bash
# k_permute with the next pair's loads in flight (variant permpipe) vs the current kernel
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02pp; mkdir -p $O
for v in base permpipe base permpipe; do
  if [ $v = base ]; then R=""; else R=paper_variants/$v; fi
  echo "== $v" >> $O/perm.txt
  PB_ROOT=$R timeout 600 python scripts/perm_bench.py >> $O/perm.txt 2>&1
done
echo done
