#!/bin/bash
# full round check: smoke, GPU tests, bench (single + batch), launch list, level-0 ncu capture
mkdir -p gpurun_out
TAG=${1:-r1c}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --workload batch --steps 10 > gpurun_out/bench_batch_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "bench batch rc=$?"
timeout 600 python bench.py --workload batch --steps 10 --opt batch_cluster=1 > gpurun_out/bench_batchcl_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "bench batch cluster rc=$?"
bash scripts/gpu_profile_round.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_batch_$TAG.csv python bench.py --workload batch --steps 1 --warmup 1 > /dev/null 2>&1; echo "batch launch list rc=$?"
