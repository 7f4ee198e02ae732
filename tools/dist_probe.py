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
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--cooldown", type=float, default=0.5, help="idle seconds before every measurement")
    p.add_argument("--rounds", type=int, default=0, help="repeat single / rank 0 / last rank this many times")
    p.add_argument("--ab", type=int, default=0,
                   help="rounds of an interleaved A/B/C of PM_OPT_UPPER_FUSED 2 / 1 / 0 (median per variant)")
    args = p.parse_args()
    n, m, W = int(args.rows), 10, args.world
    s = PartitionSolver(0)
    a, b, c, d = s.generate_device(n, 42)
    x = torch.empty_like(a)
    iface = torch.zeros(8 * W, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()

    def timed(fn):
        # B200 holds its burst clocks for ~40-50 ms of back-to-back solves, then
        # the power limit takes ~10 % (measured: 0.883 -> 0.99 ms per 8e7
        # solve); every measurement starts from an idle GPU and stays short
        import time

        torch.cuda.synchronize()
        time.sleep(args.cooldown)
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
    if args.rounds:
        res = {}
        for _ in range(args.rounds):
            res.setdefault("single", []).append(timed(lambda: s.solve_device(a, b, c, d, m=m, out=x)))
            for r in (0, W - 1):
                def one():
                    s.dist_reduce(a, b, c, d, m=m, rank=r, world=W, iface=iface[8 * r:8 * r + 8])
                    s.dist_solve(a, b, c, d, x, m=m, rank=r, world=W, iface_all=iface)
                res.setdefault(f"rank{r}", []).append(timed(one))
        out["rounds_ms"] = {k: [round(t, 4) for t in v] for k, v in res.items()}
    if args.ab:
        from paper_2501_05938_b200.solver import PM_OPT_UPPER_FUSED

        res = {}
        for _ in range(args.ab):
            for fused in (2, 1, 0):
                s.set_option(PM_OPT_UPPER_FUSED, fused)
                res.setdefault(f"single_f{fused}", []).append(timed(lambda: s.solve_device(a, b, c, d, m=m, out=x)))
                for r in (0, W - 1):
                    def one():
                        s.dist_reduce(a, b, c, d, m=m, rank=r, world=W, iface=iface[8 * r:8 * r + 8])
                        s.dist_solve(a, b, c, d, x, m=m, rank=r, world=W, iface_all=iface)
                    res.setdefault(f"rank{r}_f{fused}", []).append(timed(one))
        s.set_option(PM_OPT_UPPER_FUSED, 1)
        import statistics

        out["ab_median_ms"] = {k: round(statistics.median(v), 4) for k, v in res.items()}
        out["ab_all_ms"] = {k: [round(t, 4) for t in v] for k, v in res.items()}
    s.check()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
