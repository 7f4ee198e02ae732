#!/usr/bin/env python
"""Per-rank cost of the row-sharded solve on one GPU (a measurement tool):
rank 0 of `world` (ragged, non-last) and the last rank run pm_dist_reduce +
pm_dist_solve on 8e7 rows each; their device time (CUDA events, interface
rows exchanged through a device buffer, no collective) is compared with the
single-system solve of the same rows."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2501_05938_b200 import PartitionSolver

    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=float, default=8e7)
    p.add_argument("--world", type=int, default=2)
    p.add_argument("--reps", type=int, default=20)
    args = p.parse_args()
    n, m, W = int(args.rows), 10, args.world
    s = PartitionSolver(0)
    a, b, c, d = s.generate_device(n, 42)
    x = torch.empty_like(a)
    iface = torch.zeros(8 * W, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.reps

    out = {"rows_per_rank": n, "world": W}
    out["single_ms"] = timed(lambda: s.solve_device(a, b, c, d, m=m, out=x))
    out["single_plan"] = s.last_plan()
    for r in range(W):  # every rank's interface rows (same local rows: a solvable chain)
        s.dist_reduce(a, b, c, d, m=m, rank=r, world=W, iface=iface[8 * r:8 * r + 8])
    for r in (0, W - 1):
        def one():
            s.dist_reduce(a, b, c, d, m=m, rank=r, world=W, iface=iface[8 * r:8 * r + 8])
            s.dist_solve(a, b, c, d, x, m=m, rank=r, world=W, iface_all=iface)
        out[f"rank{r}_ms"] = timed(one)
        from paper_2501_05938_b200.solver import PM_OPT_KERNEL_TIMES

        s.set_option(PM_OPT_KERNEL_TIMES, 1)
        one()
        out[f"rank{r}_kernels"] = [(md, lv, round(t * 1e3, 1)) for (md, lv, t) in s.kernel_times()]
        s.set_option(PM_OPT_KERNEL_TIMES, 0)
        out[f"rank{r}_launches"] = s.last_launch_count
        out[f"rank{r}_plan"] = s.last_plan()
    s.check()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
