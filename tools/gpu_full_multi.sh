#!/bin/bash
# Several --set full captures of c5 batch-program kernels: pairs of "regex skip count" after tag/dtype.
#   gpurun -- bash tools/gpu_full_multi.sh tag dtype regex1 skip1 count1 [regex2 skip2 count2 ...]
set -u
TAG=$1; DT=$2; shift 2
mkdir -p gpurun_out
i=0
while [ $# -ge 3 ]; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s $2 -c $3 \
    -o gpurun_out/full_${TAG}_$i -f python tools/prof_run.py --config c5 --dtype $DT --batch 4096 --reps 0 > gpurun_out/full_${TAG}_$i.log 2>&1
  echo "full $i rc=$?"
  i=$((i+1)); shift 3
done
