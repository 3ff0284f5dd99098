# A/B: evict-first stream loads (ld.global.cs) vs L1::no_allocate + L2 evict_first policy
run() { echo "== $1 c$2 $(SSB_LIB=$PWD/$1 timeout 900 python bench.py --config $2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['fwd_avg_ms'], r['back_avg_ms'])")"; }
for r in 1 2 3; do run ab/lib_prev.so 3; run ab/lib_na.so 3; done
