for v in base JT_NO_IPERM JT_IPERM_REV; do
  if [ $v = base ]; then bash tools/gpu_prof_batch.sh ip_$v 4096; else env $v=1 bash tools/gpu_prof_batch.sh ip_$v 4096; fi
  r=$( [ $v = base ] && timeout 300 python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | tail -1 || env $v=1 timeout 300 python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | tail -1)
  echo "$v $(echo $r | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['launch_ms'])")"
done
