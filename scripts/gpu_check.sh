#!/bin/bash
# round-2 check: smoke, full GPU tests, default bench line (config 3 + c5 + e2e + cpu baseline)
mkdir -p gpurun_out
TAG=${1:-r2k}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -4 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python scripts/summarize_bench.py gpurun_out/bench_$TAG.json 2>/dev/null || tail -c 3000 gpurun_out/bench_$TAG.json
