#!/bin/bash
# --set full (with source) of launch number SKIP of kernels matching REGEX in the c5 batch program.
#   gpurun --timeout 900 -- bash tools/gpu_prof_one.sh tag regex skip [count]
set -u
TAG=$1; RE=$2; SKIP=$3; CNT=${4:-1}
mkdir -p gpurun_out
timeout 700 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT \
  -o gpurun_out/prof_${TAG} -f python tools/prof_run.py --config c5 --batch 4096 --reps 1 > gpurun_out/ncu_${TAG}.log 2>&1
echo "full rc=$?"
