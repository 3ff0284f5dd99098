#!/bin/bash
# ncu --set full of the multi-RHS kernels (config 4, 128 slices per plan), summarised on the box
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 3 --slices-per-plan 128 --no-cpu-baseline"
$CMD > gpurun_out/c4_plain.log 2>&1 || { tail gpurun_out/c4_plain.log; exit 1; }
tail -1 gpurun_out/c4_plain.log | cut -c1-200
for dir in fwd back; do
  ncu --set full --clock-control none --import-source on -k regex:"sart_${dir}_multi" -s 4 -c 1 \
      -o gpurun_out/prof_c4_$dir $CMD > gpurun_out/ncu_c4_$dir.log 2>&1
  tail -1 gpurun_out/ncu_c4_$dir.log
  ncu -i gpurun_out/prof_c4_$dir.ncu-rep --page raw --csv > gpurun_out/raw_c4_$dir.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/raw_c4_$dir.csv gpurun_out/ncu_c4_$dir.json
  rm -f gpurun_out/prof_c4_$dir.ncu-rep
done
