#!/bin/bash
# ncu launch lists (time, DRAM bytes, grid, registers) of single-tree propagations
#   gpurun -- bash tools/gpu_single_list.sh tag "c5 c4B" [dtype]
set -u
TAG=$1; CFGS=$2; DT=${3:-f32}
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread,lts__t_bytes.sum \
    --clock-control none --csv --log-file gpurun_out/single_${TAG}_${c}_${DT}.csv \
    python tools/prof_run.py --single --config $c --dtype $DT --reps 1 > /dev/null 2>&1; echo "$c rc=$?"
done
