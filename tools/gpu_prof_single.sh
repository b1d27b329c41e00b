#!/bin/bash
# Launch lists (+dram bytes) of single-tree propagations, and one full capture.
#   gpurun --timeout 1200 -- bash tools/gpu_prof_single.sh tag "c3 c4B" [full-config] [full-skip]
set -u
TAG=${1:-s01}; CONFIGS=${2:-"c3 c4B c2"}; FULLCFG=${3:-c3}; FULLSKIP=${4:-5}
mkdir -p gpurun_out
for c in $CONFIGS; do
  for dt in f32 f64; do
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread \
      --clock-control none -k regex:wave --csv --log-file gpurun_out/single_${TAG}_${c}_${dt}.csv \
      python tools/prof_run.py --single --config $c --dtype $dt --reps 1 > /dev/null 2>&1; echo "$c $dt rc=$?"
  done
done
if [ "$FULLCFG" != "none" ]; then
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wave -s $FULLSKIP -c 6 \
  -o gpurun_out/prof_${TAG}_${FULLCFG} -f python tools/prof_run.py --single --config $FULLCFG --dtype f32 --reps 1 > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "full rc=$?"
fi
