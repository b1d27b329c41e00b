#!/bin/bash
# One --set full capture of a batch-program kernel (regex, skip count) for the source/stall view.
#   gpurun -- bash tools/gpu_full_one.sh tag dtype "regex" skip
set -u
TAG=$1; DT=$2; RE=$3; SK=$4
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SK -c ${5:-1} \
  -o gpurun_out/full_$TAG -f python tools/prof_run.py --config c5 --dtype $DT --batch 4096 --reps 0 > gpurun_out/full_$TAG.log 2>&1
echo "full rc=$?"
