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
  r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(f\"{d['ms_per_step']:.4f} ms  solve {r['kernel_ms']:.4f} ({r['frac']:.3f})  reduce {r['stage1']['kernel_ms']:.4f} ({r['stage1']['frac']:.3f})  whole {r['whole_solve']['frac']:.3f}\")" 2>&1)
  echo "$lib $opts :: $r" | tee -a $OUT
done < ${CONFIGS:-scripts/sweep_configs.txt}
