#!/bin/bash
# FP32 profile: launch list of one step + full capture of the level-0 pair kernels
mkdir -p gpurun_out
TAG=${1:-f32}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --precision f32 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:warp_pair_kernel -s 2 -c 2 -o gpurun_out/prof_pair_$TAG python bench.py --precision f32 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_pair_$TAG.log 2>&1; echo "full rc=$?"
