#!/bin/bash
# batch kernels: parity tests (stream + cluster + level batch), config-4 bench lines per kernel
mkdir -p gpurun_out
TAG=${1:-r2f}
timeout 900 python -m pytest tests/test_gpu_batch_stream.py tests/test_gpu_parity.py -k "batch or stream" -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_batch_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_batch_$TAG.log
tail -3 gpurun_out/pytest_batch_$TAG.log
for opt in "batch_cluster=0" "batch_cluster=2" "batch_cluster=1"; do
  f=gpurun_out/bench_batch_${TAG}_${opt//[=,]/_}
  timeout 300 python bench.py --workload batch --opt $opt --steps 10 --warmup 3 --no-e2e --no-cpu > $f.json 2> $f.err
  echo "$opt rc=$?"; python -c "
import json; d=json.loads(open('$f.json').read().strip().splitlines()[-1]); print('$opt', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), d['roofline']['whole_step'], d.get('clocks'))"
done
