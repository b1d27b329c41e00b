#!/bin/bash
# Single-tree timings (c3, c4B, c5) for every variants/*.so.  Under gpurun.
for f in variants/*.so; do
  r=$(JT_LIB=$f timeout 300 python tools/single_bench.py c3 c4B c5 --dtypes f32 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(' '.join(f'{k}={v[\"ms\"]}' for k,v in d.items()))")
  echo "$f $r"
done
