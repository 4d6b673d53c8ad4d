#!/bin/bash
# DMMA element order A/B on one box: new rule (sorted unless sparse), old rule (any fewer tiles), never
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02pm2; mkdir -p $O
for r in 1 2; do
  timeout 600 python scripts/gate_times.py rqc 30 20 f64 5 > $O/gt_new_$r.txt 2>&1
  TSG_DMMA_PERM_ANY=1 timeout 600 python scripts/gate_times.py rqc 30 20 f64 5 > $O/gt_any_$r.txt 2>&1
  TSG_NO_DMMA_PERM=1 timeout 600 python scripts/gate_times.py rqc 30 20 f64 5 > $O/gt_none_$r.txt 2>&1
done
for v in "" "TSG_DMMA_PERM_ANY=1" "TSG_NO_DMMA_PERM=1" ""; do
  echo "== $v $(env $v timeout 600 python scripts/variant_times.py 2>&1 | tail -2 | tr '\n' ' ')" >> $O/totals.txt
done
echo done
