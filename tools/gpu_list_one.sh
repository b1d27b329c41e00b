#!/bin/bash
# ncu launch list (time, DRAM bytes, L2 hit, grid) of the c5 batch program, one dtype, extra env as VAR=val args
#   gpurun -- bash tools/gpu_list_one.sh tag dtype [VAR=val ...]
set -u
TAG=$1; DT=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__grid_size,launch__registers_per_thread \
  --clock-control none --csv --log-file gpurun_out/list_${TAG}_${DT}.csv \
  python tools/prof_run.py --config c5 --dtype $DT --batch 4096 --reps 0 > /dev/null 2>&1; echo "list $DT rc=$?"
