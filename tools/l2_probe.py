#!/usr/bin/env python
"""Effective L2 reuse capacity on this GPU (a measurement tool).

Reads one FP64 buffer of S MB with L2-cached 16-byte loads (tools/bw_probe.cu
`l2_probe`: a persistent grid, grid-stride), once to warm and then --reps
passes back to back; the repeat passes run at L2 bandwidth while L2 retains
the buffer and fall to HBM bandwidth beyond.  That retention is the budget a
config-4 design has to keep a system's rows resident between Stage 1 and
Stage 3 (the tile-stream kernel had ~80-300 MB in flight).

usage: tools/l2_probe.py [--sizes 16,32,...] [--reps 20]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "build" / "libbw_probe.so"


def main():
    import torch

    p = argparse.ArgumentParser()
    p.add_argument("--sizes", default="8,16,32,48,64,80,96,112,128,160,192,256,512,2048")
    p.add_argument("--reps", type=int, default=20)
    a = p.parse_args()
    SO.parent.mkdir(exist_ok=True)
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", str(ROOT / "tools" / "bw_probe.cu"), "-o", str(SO)], check=True)
    L = C.CDLL(str(SO))
    L.l2_probe.restype = C.c_float
    L.l2_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int]
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    out = []
    for mb in map(int, a.sizes.split(",")):
        n = mb * (1 << 20) // 8
        buf = torch.ones(n, dtype=torch.float64, device="cuda")
        best = max(n * 8 / (L.l2_probe(buf.data_ptr(), sink.data_ptr(), n, cps, 512, a.reps) / 1e3) / 1e9
                   for cps in (2, 4))
        out.append({"mb": mb, "repeat_pass_gbs": round(best, 1)})
        print(json.dumps(out[-1]), flush=True)
        del buf
    print(json.dumps({"l2_probe": out}))


if __name__ == "__main__":
    main()
