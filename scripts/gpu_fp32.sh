#!/bin/bash
# FP32: bench line and the FP32 stream sweep (Table 5 on B200)
mkdir -p gpurun_out
timeout 600 python bench.py --precision f32 --no-cpu > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err; echo "bench f32 rc=$?"; python scripts/summarize_bench.py < gpurun_out/bench_f32.json; tail -c 400 gpurun_out/bench_f32.json
timeout 2400 python tools/refit.py --reps 10 --precision f32 --out gpurun_out/refit_fp32 > gpurun_out/refit_fp32.log 2>&1; echo "refit fp32 rc=$?"
tail -25 gpurun_out/refit_fp32.log
