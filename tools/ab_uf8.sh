# K1 with 8 loads in flight per lane (UF 8) at 3 / 4 CTAs per SM vs the default (UF 4, 4 CTAs)
run() { echo "== $* $(env "$@" timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['config']['kernels']; print(d['value'], k['fwd_kernel'], r['fwd_avg_ms'], r['back_avg_ms'])")"; }
for r in 1 2; do
run SSB_LIB=$PWD/ab/lib_prev.so
run SSB_LIB=$PWD/ab/lib_u8_3.so SSB_UF_FWD=8
run SSB_LIB=$PWD/ab/lib_u8_3.so
run SSB_LIB=$PWD/ab/lib_u8_4.so SSB_UF_FWD=8
done
