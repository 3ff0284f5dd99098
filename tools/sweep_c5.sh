# config 5 K2 lane-group sweep: VS_BACK 8 (int32 fallback) vs 4 (16-bit tiles may fit)
for v in "" "SSB_VS_BACK=4" "SSB_VS_BACK=4 SSB_UF_BACK=4"; do
  echo "== $v"
  env $v timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['config']['kernels']; r=d['roofline']; print(d['value'], k['layout'], k['vs_back'], k['uf_back'], k['back_kernel'], r['fwd_avg_ms'], r['back_avg_ms'], d['e2e']['value'])"
done
