#!/bin/bash
# Round-2 final evidence on THIS build: ncu launch lists with DRAM bytes (config 3, 4 level /
# cluster / stream, 5), traffic stamped with the build hash, full captures of the level-0
# kernels, then the bench lines (which now quote the fresh traffic).
mkdir -p gpurun_out
TAG=${1:-r2f}
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M --log-file gpurun_out/launches_single_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-c5 > gpurun_out/ncu_single_$TAG.log 2>&1; echo "single rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_batch_$TAG.csv python bench.py --workload batch --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_batch_$TAG.log 2>&1; echo "batch rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_cluster_$TAG.csv python bench.py --workload batch --opt batch_cluster=1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cluster_$TAG.log 2>&1; echo "cluster rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_stream_$TAG.csv python bench.py --workload batch --opt batch_cluster=2 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_stream_$TAG.log 2>&1; echo "stream rc=$?"
timeout 600 ncu $M --log-file gpurun_out/launches_f32_$TAG.csv python bench.py --precision f32 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_f32_$TAG.log 2>&1; echo "f32 rc=$?"
timeout 900 ncu $M --log-file gpurun_out/launches_c5_$TAG.csv python bench.py --workload c5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c5_$TAG.log 2>&1; echo "c5 rc=$?"
python tools/stamp_traffic.py --single gpurun_out/launches_single_$TAG.csv --batch gpurun_out/launches_batch_$TAG.csv \
  --batch-cluster gpurun_out/launches_cluster_$TAG.csv --batch-stream gpurun_out/launches_stream_$TAG.csv \
  --f32 gpurun_out/launches_f32_$TAG.csv \
  --out gpurun_out/ncu_traffic_$TAG.json > /dev/null; echo "stamp rc=$?"
cp gpurun_out/ncu_traffic_$TAG.json profiles/ncu_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:warp_tile_kernel -s 2 -c 2 -o gpurun_out/prof_warp_$TAG python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-c5 > gpurun_out/ncu_warp_$TAG.log 2>&1; echo "full rc=$?"
# bench lines (not under a profiler)
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --precision f32 > gpurun_out/bench_f32_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "bench f32 rc=$?"
timeout 600 python bench.py --workload batch --steps 10 > gpurun_out/bench_batch_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "bench batch rc=$?"
timeout 600 python bench.py --workload batch --steps 10 --opt batch_cluster=2 --no-e2e > gpurun_out/bench_batch_stream_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "bench batch stream rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_$TAG.json 2>> gpurun_out/bench_$TAG.err; echo "bench reference rc=$?"
python - <<PY
import json
for f in ["bench_$TAG", "bench_f32_$TAG", "bench_batch_$TAG", "bench_batch_stream_$TAG", "bench_reference_$TAG"]:
    try:
        d = json.loads(open("gpurun_out/%s.json" % f).read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f, round(d.get("ms_per_step") or 0, 4), "value %.4g" % d["value"], "frac", r.get("frac"), "traffic", r.get("traffic"),
              "e2e", (d.get("e2e") or {}).get("value"), "clocks", d.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
