#!/bin/bash
# Launch list + one ncu --set full capture of the paired SART kernels (config 3 fp32).
# Each ncu command runs only after the same command exited 0 without ncu.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-large"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
# direct launches for the list: ncu drops the K1 nodes of graph replays (measured)
SSB_GRAPH=0 $CMD > gpurun_out/plain_nograph.log 2>&1 &&
SSB_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --page raw \
    $CMD > gpurun_out/launches_raw.csv 2> gpurun_out/ncu_launch.err
python tools/launch_runs.py gpurun_out/launches_raw.csv
for dir in fwd back; do
  ncu --set full --clock-control none --import-source on -k regex:"sart_${dir}_pair" -s 20 -c 2 \
      -o gpurun_out/prof_pair_$dir $CMD > gpurun_out/ncu_full_$dir.log 2>&1
  tail -2 gpurun_out/ncu_full_$dir.log
done
# summarise on the box (gpurun_out/ must stay under 64 MiB to come back)
python tools/launch_summary.py gpurun_out/launches_raw.csv gpurun_out/launches.csv \
    gpurun_out/launch_summary.txt "SSB_GRAPH=0 $CMD" && rm -f gpurun_out/launches_raw.csv
for dir in fwd back; do
  ncu -i gpurun_out/prof_pair_$dir.ncu-rep --page raw --csv > gpurun_out/raw_$dir.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/raw_$dir.csv gpurun_out/ncu_$dir.json
  rm -f gpurun_out/prof_pair_$dir.ncu-rep  # 35 MB each: summarised above
done
du -sh gpurun_out/* | sort -h | tail -5
