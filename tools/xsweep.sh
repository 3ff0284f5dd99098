for ch in 0 512 2048; do for m in 0 1 2 3; do
  echo "chunk=$ch mode=$m $(SSB_XCHUNK=$ch SSB_XMODE=$m ONLY=peer_g1 REPS=3 timeout 300 python tools/bench_exchange.py 2>&1 | tail -1)"
done; done
