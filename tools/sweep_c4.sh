#!/bin/bash
# config-4 bench line per environment variant
for spec in "$@"; do
  out=$(env $spec timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "[$spec] $(echo "$out" | python -c 'import json,sys
try:
    d=json.loads(sys.stdin.read()); print(d["value"], d["kernels"]["fwd_avg_ms"], d["kernels"]["back_avg_ms"], d["e2e"]["value"])
except Exception as e: print("FAILED", e)')"
done
