# L1 / shared-memory carveout of the paired SART kernels (smem per CTA now 2.2 KB)
for v in "" "SSB_CARVEOUT=0" "SSB_CARVEOUT=10" "SSB_CARVEOUT=25" "SSB_CARVEOUT=50"; do
  echo "== $v $(env $v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['fwd_avg_ms'], r['back_avg_ms'])")"
done
echo "== c5 $(timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['fwd_avg_ms'], r['back_avg_ms'])")"
echo "== c5 co0 $(SSB_CARVEOUT=0 timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['fwd_avg_ms'], r['back_avg_ms'])")"
