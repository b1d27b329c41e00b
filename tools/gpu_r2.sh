#!/bin/bash
# Round-2 GPU pass: parity tests, the bench line (fp64 headline + fp32), the
# self-launched multi-rank smoke, and the ncu launch list (time + DRAM bytes) of
# the fp64 and fp32 batch programs (roofline.traffic per dtype).
#   gpurun --timeout 2400 -- bash tools/gpu_r2.sh tag [skip_tests]
set -u
TAG=${1:-r2a}; SKIPT=${2:-0}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
if [ "$SKIPT" = "0" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_$TAG.json
timeout 300 python bench.py --gpus 2 --cases 1024 --batch 512 --steps 2 --no-extra --no-cpu-baseline \
  > gpurun_out/bench2_$TAG.json 2> gpurun_out/bench2_$TAG.err; echo "bench2 rc=$?"
tail -c 600 gpurun_out/bench2_$TAG.json
for DT in f64 f32; do
  timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none --csv --log-file gpurun_out/batch_${TAG}_${DT}.csv \
    python tools/prof_run.py --config c5 --dtype $DT --batch 4096 --reps 1 > /dev/null 2>&1; echo "list $DT rc=$?"
done
