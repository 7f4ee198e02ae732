#!/bin/bash
# A/B: bench sweep of a library variant against the working tree (scripts/sweep_ab.txt),
# then the GPU parity suite (TESTS=0 skips it)
mkdir -p gpurun_out
TAG=${TAG:-ab} CONFIGS=${CONFIGS:-scripts/sweep_ab.txt} bash scripts/gpu_sweep.sh
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -5 > gpurun_out/ab_tests.txt
  cat gpurun_out/ab_tests.txt
fi
