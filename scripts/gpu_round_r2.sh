#!/bin/bash
# round refresh: full round check + sanitizer (memcheck, racecheck)
bash scripts/gpu_round_full.sh ${1:-r1g}
timeout 600 python bench.py --precision f32 > gpurun_out/bench_f32_${1:-r1g}.json 2>> gpurun_out/bench_${1:-r1g}.err; echo "bench f32 rc=$?"
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
