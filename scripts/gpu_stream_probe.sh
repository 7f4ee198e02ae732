#!/bin/bash
# tile-stream kernel probe + its parity tests
mkdir -p gpurun_out
TAG=${1:-r2e}
timeout 600 python tools/stream_probe.py --reps 3 ${PROBE_SETS} > gpurun_out/probe_$TAG.log 2>&1; echo "probe rc=$?"
python - <<PY
import json
for l in open('gpurun_out/probe_$TAG.log'):
    if l.startswith('{'):
        d=json.loads(l); s=d['stats']
        print(d['variant'], d['ms'], d['GBps_40B'], d['plan'], 'cw', s['cflag_wait_frac'], 's2', s['stage2_us_each'], 'pub', s['publish_us_each'], 'tl', d.get('timeline_us_p10_50_90_99',{}).get('A_spread'))
    elif 'Error' in l or 'error' in l: print(l[:300])
PY
if [ -z "$NO_TESTS" ]; then
timeout 600 python -m pytest tests/test_gpu_batch_stream.py -q -p no:cacheprovider --timeout 120 -x > gpurun_out/pytest_stream_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stream_$TAG.log
tail -3 gpurun_out/pytest_stream_$TAG.log
fi
