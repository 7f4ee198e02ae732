import json, sys
# usage: summarize_bench.py [BENCH.json]  (stdin when no path is given)
line = (open(sys.argv[1]).read() if len(sys.argv) > 1 else sys.stdin.read()).strip().splitlines()
try:
    d = json.loads(line[-1])
except Exception:
    print("ERROR: " + " | ".join(line[-3:]))
    sys.exit(0)
r = d["roofline"]
out = f"{d['ms_per_step']:.4f} ms  solve {r.get('kernel_ms', float('nan')):.4f} ({r['frac']:.3f})"
if "stage1" in r:
    out += f"  reduce {r['stage1']['kernel_ms']:.4f} ({r['stage1']['frac']:.3f})"
if "whole_solve" in r:
    out += f"  whole {r['whole_solve']['frac']:.3f}"
print(out + f"  kernels {r.get('kernels_ms')}")
