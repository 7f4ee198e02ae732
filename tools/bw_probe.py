#!/usr/bin/env python
"""Run tools/bw_probe.cu: HBM ceilings of the level-0 access patterns
(N = 8e7 FP64 rows; read4 = Stage 1's 32 B/unknown, read4write1 = Stage 3's
40 B/unknown) over a small grid of launch shapes; prints JSON (best GB/s)."""
import ctypes as C
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "build" / "libbw_probe.so"


def main():
    import torch

    SO.parent.mkdir(exist_ok=True)
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", str(ROOT / "tools" / "bw_probe.cu"), "-o", str(SO)], check=True)
    L = C.CDLL(str(SO))
    L.bw_probe.restype = C.c_float
    L.bw_probe.argtypes = [C.c_int] + [C.c_void_p] * 5 + [C.c_int64, C.c_int, C.c_int, C.c_int]
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 80_000_000
    arrs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(5)]
    out = {}
    for kind, name, bpu in ((0, "read4", 32), (1, "read4write1", 40)):
        best = None
        for cps in (1, 2, 4, 8):
            for thr in (256, 512, 1024):
                if cps * thr > 2048:
                    continue
                ms = L.bw_probe(kind, *[a.data_ptr() for a in arrs], n, cps, thr, 20)
                if ms > 0:
                    gbs = bpu * n / (ms / 1e3) / 1e9
                    if best is None or gbs > best[0]:
                        best = (gbs, cps, thr, ms)
        out[name] = {"gbs": best[0], "ctas_per_sm": best[1], "threads": best[2], "ms": best[3],
                     "bytes_per_unknown": bpu}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
