#!/bin/bash
# time the main build and every paper_variants/* build with scripts/variant_times.py
mkdir -p gpurun_out
out=gpurun_out/variants_$(date +%H%M%S).txt
echo "== main" >> $out; timeout 300 python scripts/variant_times.py >> $out 2>&1
for v in paper_variants/*/; do echo "== $v" >> $out; PB_ROOT=$v timeout 300 python scripts/variant_times.py >> $out 2>&1; done
cat $out
