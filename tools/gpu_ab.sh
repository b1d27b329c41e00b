#!/bin/bash
# A/B bench of planner/kernel env variants on the batch workload (one line of
# space-separated VAR=value per variant in the file; the first run is the default).
#   gpurun --timeout 1800 -- bash tools/gpu_ab.sh tag dtype variants.txt [extra bench args]
set -u
TAG=$1; DT=$2; VF=$3; shift 3
mkdir -p gpurun_out
OUT=gpurun_out/ab_$TAG.txt
: > $OUT
run() {
  env "$@" timeout 300 python bench.py --dtype $DT --no-extra --no-cpu-baseline --no-e2e --steps 5 $EXTRA 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['launch_ms'], d['roofline']['frac'], d['spot_check']['max_rel_err'])" 2>&1
}
EXTRA="$*"
echo "[default] $(run JT_AB=0)" | tee -a $OUT
while read -r line; do
  [ -z "$line" ] && continue
  echo "[$line] $(run $line)" | tee -a $OUT
done < $VF
