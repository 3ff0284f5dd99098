set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for t in 1 0; do
  SSB_TILED=$t python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c3_t$t.json 2> gpurun_out/ab_c3_t$t.err
  SSB_TILED=$t python bench.py --config 2 --dtype f32 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c2_t$t.json 2>&1
  SSB_TILED=$t python bench.py --config 3 --dtype f64 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c3d_t$t.json 2>&1
done
for f in gpurun_out/ab_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().split('\n')[-1]); r=d['roofline']; print('$f', d['value'], r['fwd_avg_ms'], r['back_avg_ms'], r['frac'], d['e2e'] and d['e2e']['value'])"; done
