#!/usr/bin/env python
"""Burst vs sustained B200 throughput of one solve size (a measurement tool).

B200 holds its burst clocks for ~40-50 ms of back-to-back solves; then the
power limit costs ~10 % (0.883 -> ~0.99 ms per N = 8e7 solve).  This tool
times (a) single solves after an idle cooldown (each one alone, CUDA events)
and (b) a back-to-back run of --steps solves, and samples nvidia-smi SM
clocks / power during (b).  N = 1e9 (BASELINE config 5 on one GPU) takes
~11-12 ms per solve, so its bench steps always run in the sustained regime.

usage: tools/power_probe.py [--rows 1e9] [--steps 20] [--idle 5] [--cooldown 1.0]
"""
from __future__ import annotations

import argparse
import json
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2501_05938_b200 import PartitionSolver

    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=float, default=1e9)
    p.add_argument("--m", type=int, default=10)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--idle", type=int, default=5, help="single solves after a cooldown")
    p.add_argument("--cooldown", type=float, default=1.0)
    p.add_argument("--opt", action="append", default=[], help="NAME=VALUE: set PM_OPT_NAME")
    p.add_argument("--ktimes", action="store_true", help="kernel times of one solve after a cooldown")
    a = p.parse_args()
    n = int(a.rows)
    s = PartitionSolver(0)
    from paper_2501_05938_b200 import solver as S

    for kv in a.opt:
        k, v = kv.split("=")
        s.set_option(getattr(S, "PM_OPT_" + k.upper()), int(v))
    A, B, C, D = s.generate_device(n, 42)
    x = torch.empty_like(A)
    for _ in range(2):
        s.solve_device(A, B, C, D, m=a.m, out=x)
    torch.cuda.synchronize()

    def one():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.solve_device(A, B, C, D, m=a.m, out=x)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    idle = []
    for _ in range(a.idle):
        time.sleep(a.cooldown)
        idle.append(round(one(), 4))
    ktimes = None
    if a.ktimes:
        time.sleep(a.cooldown)
        s.set_option(S.PM_OPT_KERNEL_TIMES, 1)
        s.solve_device(A, B, C, D, m=a.m, out=x)
        ktimes = [(md, lv, round(t * 1e3, 1)) for (md, lv, t) in s.kernel_times()]
        s.set_option(S.PM_OPT_KERNEL_TIMES, 0)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
            samples.append(q)
            time.sleep(0.05)

    time.sleep(a.cooldown)
    th = threading.Thread(target=sample)
    th.start()
    per = []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.solve_device(A, B, C, D, m=a.m, out=x)
        e1.record()
        per.append((e0, e1))
    torch.cuda.synchronize()
    stop.set()
    th.join()
    s.check()
    seq = [round(e0.elapsed_time(e1), 4) for e0, e1 in per]
    bytes_ = 72.0 * n
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else None
    out = {"rows": n, "m": a.m, "opts": a.opt, "plan": s.last_plan(), "ktimes_us": ktimes, "idle_ms": idle,
           "back_to_back_ms": seq,
           "idle_best_frac": round(bytes_ / (min(idle) / 1e3) / 1e9 / peak, 4) if peak else None,
           "sustained_frac": round(bytes_ / (sorted(seq)[len(seq) // 2] / 1e3) / 1e9 / peak, 4) if peak else None,
           "smi_samples": samples[:: max(1, len(samples) // 12)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
