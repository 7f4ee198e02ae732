#!/bin/bash
# round-2 re-entry: state of the batch tile-stream kernel vs the level kernels
mkdir -p gpurun_out
TAG=${1:-r2c}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt
timeout 600 python tools/stream_probe.py --set "" --set lag=6 --set lag=12 --set warps=6 > gpurun_out/probe_$TAG.log 2>&1; echo "probe rc=$?"; cut -c1-600 gpurun_out/probe_$TAG.log | tail -6
for opt in "batch_cluster=2" "batch_cluster=0"; do
  timeout 300 python bench.py --workload batch --opt $opt --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_batch_${TAG}_${opt//[=,]/_}.json 2> gpurun_out/bench_batch_${TAG}_${opt//[=,]/_}.err
  echo "$opt rc=$?"; tail -c 1500 gpurun_out/bench_batch_${TAG}_${opt//[=,]/_}.json
done
timeout 900 python -m pytest tests/test_gpu_batch_stream.py -q -p no:cacheprovider --timeout 120 -x > gpurun_out/pytest_stream_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stream_$TAG.log
tail -3 gpurun_out/pytest_stream_$TAG.log
