# K1 row order tiles: Sb sources x Bb bins (config 3: 2048 bins per source)
for v in "" "SSB_ROWMAP_BINS=2048 SSB_ROWMAP_S=1 SSB_ROWMAP_B=32" "SSB_ROWMAP_BINS=2048 SSB_ROWMAP_S=2 SSB_ROWMAP_B=16" "SSB_ROWMAP_BINS=2048 SSB_ROWMAP_S=4 SSB_ROWMAP_B=8" "SSB_ROWMAP_BINS=2048 SSB_ROWMAP_S=2 SSB_ROWMAP_B=64" "SSB_ROWMAP_BINS=2048 SSB_ROWMAP_S=8 SSB_ROWMAP_B=4" "SSB_ROWMAP_BINS=2048 SSB_ROWMAP_S=25 SSB_ROWMAP_B=1"; do
  echo "== $v $(env $v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['fwd_avg_ms'], r['back_avg_ms'])")"
done
