#!/bin/bash
# Usage (on the GPU box via gpurun): bash tools/profile.sh <tag> [bench args...]
# 1) plain run (must exit 0), 2) ncu launch list (durations), 3) ncu --set full of one panel launch.
set -u
TAG=$1; shift
ARGS="$@"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 40 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
