#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch_stream.py -q -p no:cacheprovider --timeout 60 2>&1 | tail -2
timeout 300 python tools/sanitize_driver.py 2>&1 | tail -2
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_${tool}_r2.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_${tool}_r2.log
done
