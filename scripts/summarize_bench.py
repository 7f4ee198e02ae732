import json, sys
line = sys.stdin.read().strip().splitlines()
try:
    d = json.loads(line[-1])
except Exception:
    print("ERROR: " + " | ".join(line[-3:]))
    sys.exit(0)
r = d["roofline"]
print(f"{d['ms_per_step']:.4f} ms  solve {r['kernel_ms']:.4f} ({r['frac']:.3f})  reduce {r['stage1']['kernel_ms']:.4f} "
      f"({r['stage1']['frac']:.3f})  whole {r['whole_solve']['frac']:.3f}  kernels {r.get('kernels_ms')}")
