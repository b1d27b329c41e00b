#!/bin/bash
# Round-2 profiling pass for the batch program: A/B bench of env variants, the
# per-pass ncu launch list (JT_SPLIT_CPASS=1) and optional --set full captures.
#   gpurun --timeout 1800 -- bash tools/gpu_r2_prof.sh tag dtype "ENV1=.. ENV2=.." [full_regex] [full_skip] [full_count]
set -u
TAG=${1:-p1}; DT=${2:-f64}; VARIANTS=${3:-""}; FULLRE=${4:-""}; FSKIP=${5:-0}; FCOUNT=${6:-1}
mkdir -p gpurun_out
for V in "" $VARIANTS; do
  echo "== variant [$V]" >> gpurun_out/ab_$TAG.txt
  env $V timeout 300 python bench.py --dtype $DT --no-extra --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['launch_ms'], d['roofline']['frac'], d['spot_check']['max_rel_err'])" >> gpurun_out/ab_$TAG.txt 2>&1
done
cat gpurun_out/ab_$TAG.txt
JT_SPLIT_CPASS=1 timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none --csv --log-file gpurun_out/split_${TAG}_${DT}.csv \
  python tools/prof_run.py --config c5 --dtype $DT --batch 4096 --reps 0 > /dev/null 2>&1; echo "split list rc=$?"
if [ -n "$FULLRE" ]; then
  JT_SPLIT_CPASS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$FULLRE" -s $FSKIP -c $FCOUNT \
    -o gpurun_out/full_${TAG} -f python tools/prof_run.py --config c5 --dtype $DT --batch 4096 --reps 0 > gpurun_out/full_${TAG}.log 2>&1
  echo "full rc=$?"
fi
