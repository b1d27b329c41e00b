#!/bin/bash
# Launch list (time + DRAM bytes) of the c5 batch program (the bench step) and
# one --set full capture of its slowest kernel.
#   gpurun --timeout 900 -- bash tools/gpu_prof_batch.sh tag [batch] [full]
set -u
TAG=${1:-b01}; B=${2:-4096}; FULL=${3:-0}
mkdir -p gpurun_out
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
  --clock-control none -k regex:"wave|contract" --csv --log-file gpurun_out/batch_${TAG}.csv \
  python tools/prof_run.py --config c5 --batch $B --reps 1 > /dev/null 2>&1; echo "list rc=$?"
if [ "$FULL" = "1" ]; then
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:"contract|wave_own" -s 20 -c 6 \
    -o gpurun_out/prof_${TAG} -f python tools/prof_run.py --config c5 --batch $B --reps 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "full rc=$?"
fi
