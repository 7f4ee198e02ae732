#!/usr/bin/env python
"""Config 4 end to end (pm_solve_batch_host_f64) over staging-ring depth and
chunk size (a measurement tool): host wall clock per batch, median of --reps,
against the same-run pinned H2D bound (13.1 GB at the measured H2D rate).

usage: tools/batch_host_probe.py [--batch 4096] [--rows 100000] [--depth 2,3,4] [--chunk 10,20,40]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2501_05938_b200 import PartitionSolver, pinned_empty

    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=4096)
    p.add_argument("--rows", type=int, default=100_000)
    p.add_argument("--depth", default="0,2,3,4,6")
    p.add_argument("--chunk", default="0,10,20,40,80")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    n = a.batch * a.rows
    s = PartitionSolver(0)
    host = [pinned_empty(n) for _ in range(5)]
    for k, t in enumerate(s.generate_device(n, 42)):
        host[k][:] = t.cpu().numpy()
    torch.cuda.synchronize()
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    t0 = time.perf_counter()
    dev.copy_(torch.from_numpy(host[0]), non_blocking=True)
    torch.cuda.synchronize()
    h2d = n * 8 / (time.perf_counter() - t0) / 1e9
    bound_ms = 4 * n * 8 / h2d / 1e6
    out = {"batch": a.batch, "rows": a.rows, "h2d_gbs": round(h2d, 2), "h2d_bound_ms": round(bound_ms, 1), "runs": []}
    for depth in map(int, a.depth.split(",")):
        for chunk in map(int, a.chunk.split(",")):
            ts = []
            for _ in range(a.reps + 1):
                t0 = time.perf_counter()
                s.solve_batch_host(*host[:4], n_per_system=a.rows, depth=depth, systems_per_chunk=chunk, out=host[4])
                ts.append((time.perf_counter() - t0) * 1e3)
            ms = statistics.median(ts[1:])
            out["runs"].append({"depth": depth, "chunk": chunk, "ms": round(ms, 1),
                                "frac_of_h2d_bound": round(bound_ms / ms, 3)})
            print(json.dumps(out["runs"][-1]), flush=True)
    s.check()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
