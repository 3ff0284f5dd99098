# one bench line per BASELINE config (1 GPU), summarised
for c in "1 f64" "2 f64" "2 f32" "3 f64" "3 f32" "4 f32" "5 f32"; do
  set -- $c
  timeout 900 python bench.py --config $1 --dtype $2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg$1_$2.json 2>gpurun_out/cfg$1_$2.err
  echo "== cfg $1 $2 $(tail -1 gpurun_out/cfg$1_$2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['unit'], 'fwd', r['fwd_avg_ms'], 'back', r['back_avg_ms'], 'streamed_frac', r.get('streamed_frac'), 'e2e', d['e2e']['value'])")"
done
