#!/bin/bash
# Kernel-parameter sweep on config 3 (run under gpurun); prints one summary line per setting.
summ() { python - "$1" "$2" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f'{sys.argv[2]:40s} it/s={d["value"]:8.1f} fwd={r["fwd_avg_ms"]*1e3:6.1f}us back={r["back_avg_ms"]*1e3:6.1f}us stream={d["hbm_gbs_per_iteration_stream"]:7.1f}GB/s')
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
}
i=0
while read -r line; do
  [ -z "$line" ] && continue
  i=$((i+1))
  env $line timeout 300 python bench.py --no-cpu-baseline --no-large --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/sweep_$i.log 2>&1
  summ gpurun_out/sweep_$i.log "$line"
done
