#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:batch_stream -s 2 -c 1 python tools/stream_probe.py --reps 1 --cooldown 0.2 --set stages=1,warps=14,discard=15 > gpurun_out/ncu_stream_r3c.txt 2>&1
echo rc=$?; grep -E "duration|inst_executed|dram__bytes|issue_active|hit_rate|fp64" gpurun_out/ncu_stream_r3c.txt
