#!/bin/bash
# Round-2 artifacts on one GPU: the default bench line (config 3), the
# reference arm, GPU tests, smoke, the config-3 launch list + ncu of the pair
# kernels (tools/profile_c3.sh), and ncu summaries of the config-4 staged
# kernels and the config-1 cluster kernel (tools/profile_cfg.sh).
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
tail -1 gpurun_out/bench_full.json | cut -c1-300
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -1 gpurun_out/bench_ref.json | cut -c1-200
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
bash tools/profile_c3.sh
bash tools/profile_cfg.sh "sart_stage_kernel" c4stage 4 f32
bash tools/profile_cfg.sh "sart_cluster_pair" c1cluster 1 f64
rm -f gpurun_out/src_*.csv
du -sh gpurun_out
