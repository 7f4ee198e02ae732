#!/bin/bash
# one ncu --set full capture of a kernel (regex $1) of bench.py, tag $2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s ${SKIP:-2} -c ${COUNT:-1} -o gpurun_out/prof_$2 python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_$2.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_$2.log
