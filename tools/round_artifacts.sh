#!/bin/bash
# Round artifacts on one GPU: full bench line, reference arm, tests, launch list
# and one ncu --set full capture of the paired SART kernels (tools/profile_c3.sh).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -1 gpurun_out/bench_full.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -1 gpurun_out/bench_ref.json
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
bash tools/profile_c3.sh
# fused peer exchange on one GPU (G=1 real setup, emulated G=2/4) vs NCCL and unsharded
timeout 600 python tools/bench_exchange.py > gpurun_out/bench_exchange_c3.json 2>/dev/null; tail -1 gpurun_out/bench_exchange_c3.json
CFG=2 timeout 600 python tools/bench_exchange.py > gpurun_out/bench_exchange_c2.json 2>/dev/null; tail -1 gpurun_out/bench_exchange_c2.json
