#!/bin/bash
# --set full (with source) of the first N contraction launches of the c5 batch program.
#   gpurun --timeout 900 -- bash tools/gpu_prof_contract.sh tag [regex] [count]
set -u
TAG=${1:-c01}; RE=${2:-contract_kernel}; CNT=${3:-10}
mkdir -p gpurun_out
timeout 700 ncu --set full --clock-control none --import-source on -k regex:"$RE" -c $CNT \
  -o gpurun_out/prof_${TAG} -f python tools/prof_run.py --config c5 --batch 4096 --reps 1 > gpurun_out/ncu_${TAG}.log 2>&1
echo "full rc=$?"
