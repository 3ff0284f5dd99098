#!/bin/bash
# ncu --set full capture of one SART kernel family of the config-3 bench
# (direct launches), summarised on the box: raw page CSV, per-line source page
# (stall reasons), JSON summary.   usage: tools/profile_kernel.sh <regex> <tag> [env...]
set -u
mkdir -p gpurun_out
RE=$1; TAG=$2; shift 2
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-large"
env SSB_GRAPH=0 "$@" $CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
env SSB_GRAPH=0 "$@" ncu --set full --clock-control none --import-source on -k regex:"$RE" -s 20 -c 2 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/raw_$TAG.csv gpurun_out/ncu_$TAG.json
ls -la gpurun_out/prof_$TAG.ncu-rep
