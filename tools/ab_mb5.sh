# A/B: default build (64 registers, 4 CTAs/SM) vs a 48-register build (5 CTAs/SM)
# of the pair kernels at UF 2 (K1) and UF 2 / 4 (K2), config 3 and config 5
run() { echo "== $* $(env "$@" timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-f64 --no-large $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['config']['kernels']; print(d['value'], k['fwd_kernel'], k['back_kernel'], r['fwd_avg_ms'], r['back_avg_ms'])")"; }
for r in 1 2; do
run SSB_X=0
run SSB_LIB=$PWD/paper_1902_10559_b200/csrc/build/libsymsplit_b200_mb5.so
run SSB_LIB=$PWD/paper_1902_10559_b200/csrc/build/libsymsplit_b200_mb5.so SSB_UF_FWD=2
run SSB_LIB=$PWD/paper_1902_10559_b200/csrc/build/libsymsplit_b200_mb5.so SSB_UF_FWD=2 SSB_UF_BACK=4
done
ARGS="--config 5"
run SSB_X=0
run SSB_LIB=$PWD/paper_1902_10559_b200/csrc/build/libsymsplit_b200_mb5.so SSB_UF_FWD=2
run SSB_LIB=$PWD/paper_1902_10559_b200/csrc/build/libsymsplit_b200_mb5.so SSB_UF_FWD=2 SSB_UF_BACK=4
