#!/bin/bash
# round 2: new C-ABI collective tests + stream-count re-sweeps (30 reps) for the anchored re-fit
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "solve_dist or dist_caller or mixed_precision" > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log; tail -5 gpurun_out/pytest_r2b.log
timeout 900 python tools/refit.py --reps 30 --stream-mode 0 --out gpurun_out/refit_pooled > gpurun_out/refit_pooled.log 2>&1; echo "pooled rc=$?"
timeout 900 python tools/refit.py --reps 20 --stream-mode 1 --out gpurun_out/refit_per_solve > gpurun_out/refit_per_solve.log 2>&1; echo "per-solve rc=$?"
timeout 900 python tools/refit.py --reps 20 --precision f32 --out gpurun_out/refit_fp32 > gpurun_out/refit_fp32.log 2>&1; echo "fp32 rc=$?"
tail -3 gpurun_out/refit_*.log
