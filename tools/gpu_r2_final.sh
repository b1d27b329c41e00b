#!/bin/bash
# Round-2 closing pass: GPU tests, the bench line, the 2-rank self-launch smoke,
# ncu launch lists of the batch step (both dtypes) and of the single trees, and
# one --set full capture of the top fp64 kernel (the paired hub pass).
#   gpurun --timeout 3000 -- bash tools/gpu_r2_final.sh tag
set -u
TAG=${1:-r2c}
bash tools/gpu_r2.sh $TAG
bash tools/gpu_single_list.sh $TAG "c3 c4B c5" f32
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_rowi -s 7 -c 1 \
  -o gpurun_out/full_${TAG}_paired -f python tools/prof_run.py --config c5 --dtype f64 --batch 4096 --reps 0 \
  > gpurun_out/full_${TAG}_paired.log 2>&1; echo "full rc=$?"
