# config 3 fp64: default (4 CTAs/SM, UF_FWD 2) vs 3 CTAs/SM builds with UF_FWD 4
run() { echo "== $* $(env "$@" timeout 900 python bench.py --config 3 --dtype f64 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['config']['kernels']; print(d['value'], k['fwd_kernel'], k['back_kernel'], r['fwd_avg_ms'], r['back_avg_ms'])")"; }
for r in 1 2; do
run SSB_LIB=$PWD/paper_1902_10559_b200/libsymsplit_b200.so
run SSB_LIB=$PWD/ab/lib_mb3.so SSB_UF_FWD=4
run SSB_LIB=$PWD/ab/lib_mb3.so SSB_UF_FWD=4 SSB_UF_BACK=4
run SSB_LIB=$PWD/ab/lib_mb3.so
done
