#!/bin/bash
# Single-tree A/B: GPU tests (optional), then the single-tree table under each env variant.
#   gpurun --timeout 1500 -- bash tools/gpu_single_ab.sh tag "c1 c2 c4M" variants.txt [run_tests]
set -u
TAG=$1; CFGS=$2; VF=$3; TESTS=${4:-1}
mkdir -p gpurun_out
if [ "$TESTS" = "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log; tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
OUT=gpurun_out/single_$TAG.txt
: > $OUT
echo "[default]" >> $OUT; timeout 300 python tools/single_bench.py $CFGS >> $OUT 2>&1
while read -r line; do
  [ -z "$line" ] && continue
  echo "[$line]" >> $OUT; env $line timeout 300 python tools/single_bench.py $CFGS >> $OUT 2>&1
done < $VF
cat $OUT | python -c "
import sys,json,re
txt=sys.stdin.read()
for blk in re.split(r'^(\[.*\])$', txt, flags=re.M)[1:]:
    if blk.startswith('['): print(blk); continue
    try:
        d=json.loads(blk[blk.index('{'):])
        print('  '+'  '.join(f\"{k}:{v['ms']}\" for k,v in d.items()))
    except Exception as e: print('  parse error', blk[-300:])
"
