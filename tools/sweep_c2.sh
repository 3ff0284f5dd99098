#!/bin/bash
# config-2 bench line (device it/s, e2e, persistent kernel) per environment variant
#   usage: tools/sweep_c2.sh <dtype> "ENV=.. ENV=.." ...
DT=$1; shift
for spec in "$@"; do
  echo "[$spec] $(env $spec timeout 300 python bench.py --config 2 --dtype $DT --steps 20 --warmup 3 --no-cpu-baseline --no-f64 --no-large 2>&1 | tail -1 | python -c 'import json,sys
try:
    d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["config"]["kernels"]["persistent_kernel"])
except Exception as e: print("FAILED", e)')"
done
