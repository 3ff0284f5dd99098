"""Run the config-3 bench once per environment variant and print one summary
line each (it/s, K1/K2 event times, kernel names, ring geometry).
usage: python tools/sweep_env.py "A=1 B=2" "A=0" ...   (run under gpurun)"""
import json
import os
import subprocess
import sys

base = [sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-large"]
extra = os.environ.get("SWEEP_ARGS", "").split()
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run(base + extra, env=env, capture_output=True, text=True, timeout=600)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if r.returncode != 0 or not line:
        print(f"{spec:60s} FAILED rc={r.returncode} {r.stderr[-400:]}", flush=True)
        continue
    d = json.loads(line[-1])
    k = d["config"].get("kernels", {})
    rf = d["roofline"]
    print(f"{spec:60s} {d['value']:9.1f} it/s  fwd {rf.get('fwd_avg_ms', 0) * 1e3:6.1f} us  "
          f"back {rf.get('back_avg_ms', 0) * 1e3:6.1f} us  {k.get('fwd_kernel', '')} | "
          f"{k.get('back_kernel', '')} stages={k.get('ring_stages')} chunks={k.get('ring_chunks')} "
          f"slot={k.get('ring_slot_bytes')} layout={k.get('layout')}", flush=True)
