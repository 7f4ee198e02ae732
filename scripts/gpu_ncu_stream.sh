#!/bin/bash
# ncu DRAM bytes / IPC / instructions of the tile-stream kernel per run-ahead setting ($VARIANTS)
mkdir -p gpurun_out
for v in ${VARIANTS:-lag=516 lag=260 lag=259}; do
timeout 300 ncu --metrics gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:batch_stream -s 2 -c 1 python tools/stream_probe.py --reps 1 --cooldown 0.2 --set $v > gpurun_out/ncu_stream_$v.txt 2>&1
echo "$v rc=$?"; grep -E "duration|inst_executed|dram__bytes|hit_rate" gpurun_out/ncu_stream_$v.txt
done
