#!/bin/bash
# row-sharded fused upper levels: parity tests + per-rank probe
mkdir -p gpurun_out
TAG=${1:-r2g}
timeout 900 python -m pytest tests/test_gpu_parity.py -k "dist" -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_dist_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist_$TAG.log
tail -15 gpurun_out/pytest_dist_$TAG.log
python tools/dist_probe.py --world 2 > gpurun_out/dist_probe_$TAG.json 2>&1; cat gpurun_out/dist_probe_$TAG.json | cut -c1-900
