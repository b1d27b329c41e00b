#!/bin/bash
# Bench every variants/*.so on the batch workload (program ms).  Under gpurun.
for f in variants/*.so; do
  r=$(JT_LIB=$f timeout 300 python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['launch_ms'], d['spot_check_max_rel_err'])")
  echo "$f $r"
done
