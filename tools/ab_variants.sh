# A/B of compile-time variants of sart.cu (make -C paper_1902_10559_b200/csrc variant NAME=.. DEFS=..):
# usage: bash tools/ab_variants.sh "<bench args>" name1 name2 ...   (default build first)
ARGS="$1"; shift
run() { echo "== $* $(env "$@" timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-f64 --no-large $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['config']['kernels']; print(d['value'], k['fwd_kernel'], k['back_kernel'], r['fwd_avg_ms'], r['back_avg_ms'])")"; }
for r in 1 2; do
run SSB_X=0
for n in "$@"; do run SSB_LIB=$PWD/paper_1902_10559_b200/csrc/build/libsymsplit_b200_$n.so; done
done
