# multi-RHS (config 4) measurements: 128 and 256 slices per plan; multi parity tests
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "multi" 2>&1 | tail -1
for r in 1 2; do for spp in 128 256; do
  echo "== spp $spp $(timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --slices-per-plan $spp 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(d['value'], k['fwd_avg_ms'], k['back_avg_ms'])")"
done; done
