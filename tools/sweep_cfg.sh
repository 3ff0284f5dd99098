#!/bin/bash
# usage: tools/sweep_cfg.sh CONFIG DTYPE "ENV1" "ENV2" ...  -> one summary line per variant
C=$1; D=$2; shift 2
for spec in "$@"; do
  out=$(env $spec timeout 300 python bench.py --config $C --dtype $D --steps 20 --warmup 3 --no-cpu-baseline --no-f64 --no-large 2>/dev/null | tail -1)
  echo "cfg$C $D [$spec] $(echo "$out" | python -c 'import json,sys
try:
    d=json.loads(sys.stdin.read()); k=d["config"].get("kernels",{}); print(d["value"], d["e2e"]["value"], k.get("persistent_grid"))
except Exception as e: print("FAILED", e)')"
done
