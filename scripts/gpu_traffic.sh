#!/bin/bash
# ncu launch lists (time + DRAM bytes) of one bench step per workload on THIS build,
# then stamp profiles/ncu_traffic.json with the build hash (tools/stamp_traffic.py).
mkdir -p gpurun_out
TAG=${1:-r2}
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M --log-file gpurun_out/launches_single_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-c5 > gpurun_out/ncu_single_$TAG.log 2>&1; echo "single rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_batch_$TAG.csv python bench.py --workload batch --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_batch_$TAG.log 2>&1; echo "batch rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_cluster_$TAG.csv python bench.py --workload batch --opt batch_cluster=1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cluster_$TAG.log 2>&1; echo "cluster rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_c5_$TAG.csv python bench.py --workload c5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c5_$TAG.log 2>&1; echo "c5 rc=$?"
python tools/stamp_traffic.py --single gpurun_out/launches_single_$TAG.csv --batch gpurun_out/launches_batch_$TAG.csv \
  --batch-cluster gpurun_out/launches_cluster_$TAG.csv --out gpurun_out/ncu_traffic_$TAG.json
