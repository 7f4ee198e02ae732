#!/bin/bash
# configuration sweep: bench (device-resident only) per library variant / option set
mkdir -p gpurun_out
OUT=gpurun_out/sweep_${TAG:-x}.txt
: > $OUT
while read -r lib opts; do
  [ -z "$lib" ] && continue
  args=""
  for o in $opts; do args="$args --opt $o"; done
  if [ "$lib" = "default" ]; then export -n PM_LIB_PATH; unset PM_LIB_PATH; else export PM_LIB_PATH=$lib; fi
  r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu ${BENCH_EXTRA} $args 2>&1 | python scripts/summarize_bench.py)
  echo "$lib $opts :: $r" | tee -a $OUT
done < ${CONFIGS:-scripts/sweep_configs.txt}
