#!/bin/bash
# A/B an environment switch on the batch bench, alternating runs on one box:
#   gpurun -- bash tools/ab_env.sh JT_NO_INTERLEAVE=1 [reps]
ALT=$1; N=${2:-2}
one() { env "$@" timeout 300 python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | tail -1 |
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['launch_ms'])"; }
for r in $(seq $N); do echo "base $(one JT_AB=0)"; echo "$ALT $(one $ALT)"; done
