#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_cluster -s 3 -c 1 -o gpurun_out/prof_batch_cl8 python bench.py --workload batch --steps 1 --warmup 3 --opt batch_cluster_size=8 --opt batch_warps=14 > gpurun_out/ncu_batch.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_cluster -s 3 -c 1 -o gpurun_out/prof_batch_cl6 python bench.py --workload batch --steps 1 --warmup 3 --opt batch_cluster_size=6 --opt batch_warps=12 --opt batch_l2_mb=100 >> gpurun_out/ncu_batch.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_batch.log
