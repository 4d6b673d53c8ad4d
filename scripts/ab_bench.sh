#!/bin/bash
# A/B on one box: bench.py device step with env setting A vs B, alternated 3 times
# usage: ab_bench.sh "ENV=a" "ENV=b"
mkdir -p gpurun_out
for i in 1 2 3; do
  for cfg in "$1" "$2"; do
    v=$(env $cfg python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-aux 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f qft %.4f rqc %.4f clk %s' % (d['value'], d['per_circuit_s']['qft30'], d['per_circuit_s']['rqc30'], d['clocks']['sm_mhz']))")
    echo "$cfg: $v"
  done
done
