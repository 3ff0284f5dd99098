# multi-RHS K1 column bands (SSB_BANDS) on config 4
for b in 1 2 3 4; do
  echo "== bands $b $(SSB_BANDS=$b timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(d['value'], k['fwd_avg_ms'], k['back_avg_ms'])")"
done
for spp in 64 256; do
  echo "== spp $spp $(timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --slices-per-plan $spp 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(d['value'], k['fwd_avg_ms'], k['back_avg_ms'])")"
done
