# one bench line per BASELINE config (1 GPU), summarised; the CPU baseline of
# each config runs in its own line (configs 1-4; config 5's oracle needs ~40 GB
# and minutes, so its line skips it)
mkdir -p gpurun_out
for c in "1 f64" "2 f64" "2 f32" "3 f64" "3 f32" "4 f32" "5 f32"; do
  set -- $c
  extra="--no-f64 --no-large"
  [ "$1" = "5" ] && extra="$extra --no-cpu-baseline"
  timeout 1200 python bench.py --config $1 --dtype $2 --steps 10 --warmup 3 $extra > gpurun_out/cfg$1_$2.json 2>gpurun_out/cfg$1_$2.err
  echo "== cfg $1 $2 $(tail -1 gpurun_out/cfg$1_$2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; cb=d.get('cpu_baseline') or {}; print(d['value'], d['unit'], 'fwd', r.get('fwd_avg_ms'), 'back', r.get('back_avg_ms'), 'frac', r.get('frac'), 'e2e', d['e2e']['value'], 'cpu', cb.get('value'))")"
done
