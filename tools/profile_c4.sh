#!/bin/bash
# ncu --set full of the multi-RHS kernels (config 4, 128 slices per plan)
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 1 --slices-per-plan 128"
$CMD > gpurun_out/c4_plain.log 2>&1 || { tail gpurun_out/c4_plain.log; exit 1; }
tail -1 gpurun_out/c4_plain.log | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:'sart_fwd_multi' -s 2 -c 1 \
    -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4.log 2>&1
tail -1 gpurun_out/ncu_c4.log
