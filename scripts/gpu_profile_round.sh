#!/bin/bash
# Round profile: ncu launch list of one bench step + full capture of the level-0 kernels
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:warp_tile_kernel -s 2 -c 2 -o gpurun_out/prof_warp_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_warp_$TAG.log 2>&1; echo "full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upper_fused_kernel -s 1 -c 1 -o gpurun_out/prof_upper_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_upper_$TAG.log 2>&1; echo "upper full rc=$?"
