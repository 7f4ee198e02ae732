#!/bin/bash
# end-of-round check: smoke, full GPU suite, bench lines (FP64, FP32, batch)
mkdir -p gpurun_out
TAG=${1:-final}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --precision f32 > gpurun_out/bench_f32_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "f32 rc=$?"
timeout 600 python bench.py --workload batch --steps 10 > gpurun_out/bench_batch_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "batch rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "ref rc=$?"
