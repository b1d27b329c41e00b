#!/bin/bash
# ncu launch list (time, DRAM bytes, L2 hit) of the c5 batch program, both dtypes
#   gpurun -- bash tools/gpu_list_r2.sh tag
set -u
TAG=$1
mkdir -p gpurun_out
for DT in f64 f32; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__grid_size \
    --clock-control none --csv --log-file gpurun_out/list_${TAG}_${DT}.csv \
    python tools/prof_run.py --config c5 --dtype $DT --batch 4096 --reps 1 > /dev/null 2>&1; echo "list $DT rc=$?"
done
