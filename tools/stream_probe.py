#!/usr/bin/env python
"""Probe the batch tile-stream kernel (PM_OPT_BATCH_CLUSTER = 2) on one GPU:
time one config-4 batch (4096 x 1e5, m = 10 by default) for every
--set "lag=..,warps=..,stages=..,discard=.." variant and print the kernel's
clock64 diagnostics (PM_OPT_BATCH_STATS) next to the CUDA-event time.

usage: tools/stream_probe.py [--batch 4096] [--rows 100000] [--set lag=4] [--set lag=8,warps=6] ...
"""
from __future__ import annotations

import argparse
import json
import time
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2501_05938_b200 import PartitionSolver  # noqa: E402
from paper_2501_05938_b200 import solver as S  # noqa: E402

OPTS = {"lag": S.PM_OPT_BATCH_LAG, "warps": S.PM_OPT_BATCH_WARPS, "stages": S.PM_OPT_BATCH_STAGES,
        "discard": S.PM_OPT_BATCH_DISCARD, "ctas": S.PM_OPT_MAX_CTAS, "kernel": S.PM_OPT_BATCH_CLUSTER}


def main():
    import torch

    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=4096)
    p.add_argument("--rows", type=int, default=100_000)
    p.add_argument("--m", type=int, default=10)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--cooldown", type=float, default=1.0, help="idle seconds before every variant")
    p.add_argument("--set", action="append", default=[])
    p.add_argument("--timeline", action="store_true", help="per-system timeline percentiles")
    p.add_argument("--trace", default="", help="save the sample warps' job traces (npz)")
    a = p.parse_args()
    sv = PartitionSolver(0)
    n = a.batch * a.rows
    A, B, Cc, D = sv.generate_device(n, 42)
    x = torch.empty_like(B)
    variants = a.set or [""]
    for var in variants:
        kv = {"kernel": 2}
        for item in filter(None, var.split(",")):
            k, v = item.split("=")
            kv[k] = int(v)
        for k, v in kv.items():
            sv.set_option(OPTS[k], v)
        # every variant from an idle GPU: back-to-back launches pass B200's
        # burst window (~40-50 ms) and run ~10 % slower under its power limit
        torch.cuda.synchronize()
        time.sleep(a.cooldown)
        for _ in range(2):
            sv.solve_batch_device(A, B, Cc, D, n_per_system=a.rows, m=a.m, out=x)
        sv.check()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            sv.solve_batch_device(A, B, Cc, D, n_per_system=a.rows, m=a.m, out=x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        sv.check()
        sv.set_option(S.PM_OPT_BATCH_STATS, 1)
        sv.solve_batch_device(A, B, Cc, D, n_per_system=a.rows, m=a.m, out=x)
        st = sv.batch_stream_stats()
        sv.set_option(S.PM_OPT_BATCH_STATS, 0)
        plan = sv.last_batch_plan()
        sv.check()
        out = {"variant": var or "default", "ms": round(ms, 4),
               "GBps_40B": round(40 * n / (ms / 1e3) / 1e9, 1), "plan": plan.get("stream") or plan["kernel"]}
        cw = max(1, st["compute_cyc"])
        cc = max(1, st["control_cyc"])
        out["stats"] = {
            "cflag_wait_frac": round(st["cflag_wait_cyc"] / cw, 4), "cflag_waits": st["cflag_waits"],
            "mbox_wait_frac": round(st["mbox_wait_cyc"] / cw, 4),
            "stage_wait_frac": round(st["stage_wait_cyc"] / cw, 4),
            "ctl_idle_frac": round(st["ctl_idle"] / max(1, st["ctl_iters"]), 4), "ctl_iters": st["ctl_iters"],
            "stage2_frac": round(st["stage2_cyc"] / cc, 4), "stage2_n": st["stage2_n"],
            "stage2_us_each": round(st["stage2_cyc"] / max(1, st["stage2_n"]) / 1965.0, 3),
            "publish_frac": round(st["publish_cyc"] / cc, 4),
            "publish_us_each": round(st["publish_cyc"] / max(1, st["ctl_iters"] - st["ctl_idle"]) / 1965.0, 3),
            "a_jobs": st["a_jobs"], "c_jobs": st["c_jobs"],
            "queue_us_each": round(st["queue_ns"] / max(1, st["stage2_n"]) / 1e3, 3),
            "s2_latency_us_each": round(st["s2_latency_ns"] / max(1, st["stage2_n"]) / 1e3, 3)}
        if a.timeline:
            import numpy as np

            tl = sv.batch_stream_timeline(a.batch).astype(np.float64)
            t0 = tl[0].min()
            tl = (tl - t0) / 1e3  # us since the first Stage-1 start
            q = lambda v: [round(float(np.percentile(v, p)), 2) for p in (10, 50, 90, 99)]
            out["timeline_us_p10_50_90_99"] = {
                "A_spread": q(tl[1] - tl[0]), "publish_delay": q(tl[2] - tl[1]), "stage2": q(tl[3] - tl[2]),
                "C_wait_from_first_C": q(np.maximum(0, tl[3] - tl[4])), "flag_minus_firstA": q(tl[3] - tl[0]),
                "firstC_minus_firstA": q(tl[4] - tl[0])}
            mid = a.batch // 2
            out["timeline_sample_us"] = {str(s): [round(float(v), 1) for v in tl[:, s]]
                                         for s in (0, 1, 2, 3, 4, mid, mid + 1, a.batch - 1)}
        if a.trace:
            import numpy as np

            tr, ctl, wsum = sv.batch_stream_traces(a.batch)
            t0 = int(sv.batch_stream_timeline(a.batch)[0].min())
            np.savez(a.trace, tr=tr, ctl=ctl, t0=t0, wsum=wsum)
        print(json.dumps(out), flush=True)
        for k in kv:
            sv.set_option(OPTS[k], 0 if k != "discard" else 15)


if __name__ == "__main__":
    main()
