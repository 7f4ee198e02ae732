#!/bin/bash
# batch tile-stream kernel: parity tests, then config-4 bench lines (stream vs level vs cluster)
mkdir -p gpurun_out
TAG=${1:-s1}
timeout 900 python -m pytest tests/test_gpu_batch_stream.py -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_stream_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stream_$TAG.log
tail -15 gpurun_out/pytest_stream_$TAG.log
for opt in "batch_cluster=2" "batch_cluster=0" ${EXTRA_OPTS}; do
  timeout 300 python bench.py --workload batch --opt $opt --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_batch_${TAG}_${opt//[=,]/_}.json 2> gpurun_out/bench_batch_${TAG}_${opt//[=,]/_}.err
  echo "$opt rc=$?"; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_batch_${TAG}_${opt//[=,]/_}.json').read().strip().splitlines()[-1]); print('$opt', round(d['ms_per_step'],3), 'ms', d['roofline']['frac'], d['roofline'].get('kernel','')[:40], d.get('clocks'))" 2>&1 | tail -1
done
