#!/bin/bash
# batch cluster kernel: parity tests, bench of config 4, plan sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider --timeout 300 -k "batch_cluster" > gpurun_out/pytest_batch.log 2>&1; echo "pytest batch rc=$?" >> gpurun_out/pytest_batch.log
tail -15 gpurun_out/pytest_batch.log
while read -r o; do
  echo "== $o"; timeout 300 python bench.py --workload batch --steps 10 --warmup 3 $o > gpurun_out/bb.json 2> gpurun_out/bb.err; tail -1 gpurun_out/bb.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['ms_per_step'],4), 'ms', '%.3g'%d['value'], 'frac', round(r['frac'],3), r['kernel_ms'], d['config']['cluster_plan'])" || tail -3 gpurun_out/bb.err
done < ${BATCH_CONFIGS:-scripts/batch_configs.txt}
