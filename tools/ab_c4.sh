# A/B of the multi-RHS kernels: previous commit's library (ab/lib_old.so) vs the tree's
for r in 1 2; do
for lib in ab/lib_old.so paper_1902_10559_b200/libsymsplit_b200.so; do
  echo "== $lib $(SSB_LIB=$PWD/$lib SSB_BANDS=1 timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(d['value'], k['fwd_avg_ms'], k['back_avg_ms'])")"
done; done
