#!/bin/bash
# bench lines (config 3 FP64 / FP32, config 4 level + cluster), launch lists, level-0 ncu capture
mkdir -p gpurun_out
TAG=${1:-r1h}
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --workload batch --steps 10 > gpurun_out/bench_batch_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "batch rc=$?"
timeout 600 python bench.py --workload batch --steps 10 --opt batch_cluster=1 > gpurun_out/bench_batchcl_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "batch cluster rc=$?"
timeout 600 python bench.py --precision f32 > gpurun_out/bench_f32_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "f32 rc=$?"
bash scripts/gpu_profile_round.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_batch_$TAG.csv python bench.py --workload batch --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "batch launch list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_f32_$TAG.csv python bench.py --precision f32 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "f32 launch list rc=$?"
