#!/bin/bash
# iteration loop on the GPU box: tests, bench, launch list, one ncu capture
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 5 -c 5 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
