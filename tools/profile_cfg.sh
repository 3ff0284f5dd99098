#!/bin/bash
# ncu --set full capture of one kernel family of a given config's bench
# (graph replay), raw + source pages and a JSON summary.
#   usage: tools/profile_cfg.sh <regex> <tag> <config> <dtype> [env...]
set -u
mkdir -p gpurun_out
RE=$1; TAG=$2; CFG=$3; DT=$4; shift 4
CMD="python bench.py --config $CFG --dtype $DT --steps 2 --warmup 3 --no-cpu-baseline --no-f64 --no-large"
env "$@" $CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
env "$@" ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:"$RE" -s 2 -c ${NCU_COUNT:-1} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/raw_$TAG.csv gpurun_out/ncu_$TAG.json
rm -f gpurun_out/prof_$TAG.ncu-rep
