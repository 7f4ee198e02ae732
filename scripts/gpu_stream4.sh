#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-s7}
timeout 600 python tools/stream_probe.py ${PROBE_SETS:---set ""} > gpurun_out/probe_$TAG.log 2>&1; echo "probe rc=$?"; python -c "
import json
for l in open('gpurun_out/probe_$TAG.log'):
  if l.startswith('{'):
    d=json.loads(l); s=d['stats']; print(d['variant'], d['ms'], 'cflag', s['cflag_wait_frac'], 'waits', s['cflag_waits'], 's2us', s['stage2_us_each'])
"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batch_stream -s 2 -c 1 -o gpurun_out/prof_stream_$TAG python tools/stream_probe.py --reps 1 > gpurun_out/ncu_stream_$TAG.log 2>&1; echo "ncu rc=$?"
timeout 600 python -m pytest tests/test_gpu_batch_stream.py -q -p no:cacheprovider --timeout 120 -x > gpurun_out/pytest_stream_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stream_$TAG.log
tail -3 gpurun_out/pytest_stream_$TAG.log
