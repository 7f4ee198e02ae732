#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/refit.py --reps 10 --out gpurun_out/refit_pooled > gpurun_out/refit_pooled.log 2>&1; echo "pooled rc=$?"
timeout 1500 python tools/refit.py --reps 10 --stream-mode 1 --out gpurun_out/refit_percall > gpurun_out/refit_percall.log 2>&1; echo "percall rc=$?"
tail -30 gpurun_out/refit_pooled.log
