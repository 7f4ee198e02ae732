#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2d}
timeout 600 python tools/stream_probe.py --reps 3 ${PROBE_SETS} > gpurun_out/probe_$TAG.log 2>&1; echo "probe rc=$?"; cut -c1-1200 gpurun_out/probe_$TAG.log | grep -v "^$" | tail -12
