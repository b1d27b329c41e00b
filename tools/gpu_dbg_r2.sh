mkdir -p gpurun_out
for cfg in "c2 f64 2048" "c2 f32 2048" "c4M f64 2048" "c4M f32 512"; do
  echo "== $cfg" >> gpurun_out/dbg1.txt
  timeout 300 python tools/batch_debug.py $cfg >> gpurun_out/dbg1.txt 2>&1
done
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python tools/batch_debug.py c2 f64 2048 > gpurun_out/dbg1_san.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tiny -c 1 -o gpurun_out/tiny_c1 -f python tools/prof_run.py --single --config c1 --dtype f32 --reps 1 > gpurun_out/tiny_c1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tiny -c 1 -o gpurun_out/tiny_c4M -f python tools/prof_run.py --single --config c4M --dtype f32 --reps 1 > gpurun_out/tiny_c4M.log 2>&1
