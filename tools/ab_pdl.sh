# A/B: previous build vs bounds prefetched before cudaGridDependencySynchronize
run() { echo "== $1 c$2 $(SSB_LIB=$PWD/$1 timeout 900 python bench.py --config $2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['fwd_avg_ms'], r['back_avg_ms'], d['e2e']['value'])")"; }
for r in 1 2 3; do
  for c in 3 2 1; do run ab/lib_prev.so $c; run ab/lib_pf.so $c; done
done
