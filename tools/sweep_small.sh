# configs 1-2 after the lane-group widening rule; layout tests
timeout 600 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
run() { echo "== $* $(env "${@:3}" timeout 900 python bench.py --config $1 --dtype $2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['config']['kernels']; print(d['value'], k['fwd_kernel'], k['back_kernel'], k['fwd_blocks'], k['back_blocks'], r['fwd_avg_ms'], r['back_avg_ms'])")"; }
for c in "1 f64" "2 f32" "3 f32"; do set -- $c; run $1 $2 X=1; done
