#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-s2}
timeout 600 python tools/stream_probe.py --set "" --set lag=8 --set lag=16 --set lag=8,discard=0 --set lag=8,stages=1 > gpurun_out/probe_$TAG.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe_$TAG.log | tail -12
timeout 900 python -m pytest tests/test_gpu_batch_stream.py -q -p no:cacheprovider --timeout 120 -x > gpurun_out/pytest_stream_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stream_$TAG.log
tail -25 gpurun_out/pytest_stream_$TAG.log
