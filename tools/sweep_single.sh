# single-system tiled plan (one folded system of config 3: the per-rank plan at N = 2)
for v in "X=1" "SSB_VS_FWD=8" "SSB_VS_FWD=32" "SSB_VS_BACK=4" "SSB_VS_BACK=16" "SSB_UF_FWD=2" "SSB_UF_BACK=2" "SSB_VS_FWD=8 SSB_VS_BACK=8" "SSB_VS_FWD=8 SSB_UF_BACK=2"; do
  echo "== $v $(env $v timeout 600 python tools/bench_single.py 2>/dev/null | tail -1)"
done
