#!/bin/bash
# Launch lists (time + DRAM bytes) of the c5 batch program (the bench step),
# with and without the contraction passes.
#   gpurun --timeout 900 -- bash tools/gpu_prof_batch.sh tag
set -u
TAG=${1:-b01}
mkdir -p gpurun_out
for v in CONTRACT JT_NO_CONTRACT; do
  env $v=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none -k regex:"wave|contract" --csv --log-file gpurun_out/batch_${TAG}_${v}.csv \
    python tools/prof_run.py --config c5 --reps 1 > /dev/null 2>&1; echo "$v rc=$?"
done
