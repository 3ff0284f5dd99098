# config 5 lane-group / unroll sweep (K2 narrowed to 4 lanes with 16-bit offsets)
for v in "" "SSB_VS_FWD=32" "SSB_VS_FWD=8" "SSB_UF_FWD=2" "SSB_VS_FWD=32 SSB_UF_FWD=2" "SSB_STREAM_CS=0" "SSB_L2WIN=1"; do
  echo "== $v $(env $v timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['config']['kernels']; r=d['roofline']; print(d['value'], k['fwd_kernel'], k['back_kernel'], r['fwd_avg_ms'], r['back_avg_ms'], r['streamed_frac'])")"
done
