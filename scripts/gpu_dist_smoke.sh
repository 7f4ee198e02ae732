#!/bin/bash
# two ranks sharing cuda:0 over gloo: exercises bench.py's row-sharded path
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --rows-per-gpu 4e6 --dist-backend gloo --same-device --no-e2e > gpurun_out/dist_smoke.json 2> gpurun_out/dist_smoke.err; echo "dist rc=$?"
cat gpurun_out/dist_smoke.json | cut -c1-600; tail -5 gpurun_out/dist_smoke.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; echo "ref rc=$?"; cut -c1-400 gpurun_out/ref_arm.json
