#!/bin/bash
# compute-sanitizer memcheck + racecheck over small trees and a small batch
# (race detection / failure detection on device).  Run under gpurun.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
