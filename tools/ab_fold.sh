# A/B of the fold's fill-pass stores: plain vs evict-last L2 policy (SSB_FOLD_EVICT_LAST build)
for r in 1 2; do for lib in ab/lib_prev.so ab/lib_el.so; do
  echo "== $lib $(SSB_LIB=$PWD/$lib REPS=3 timeout 300 python tools/trace_e2e.py 3 2>&1 | grep -E 'verify_symmetry|call 2' | tail -2 | tr '\n' ' ')"
done; done
SSB_LIB=$PWD/ab/lib_el.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "split or fold or build" 2>&1 | tail -1
