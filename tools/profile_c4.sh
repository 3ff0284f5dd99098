#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 1"
$CMD > gpurun_out/c4_plain.log 2>&1 || { tail gpurun_out/c4_plain.log; exit 1; }
tail -1 gpurun_out/c4_plain.log
ncu --set full --clock-control none -k regex:'sart_(fwd|back)_multi' -s 10 -c 2 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4.log 2>&1
tail -1 gpurun_out/ncu_c4.log
