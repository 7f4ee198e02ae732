#!/usr/bin/env python
"""Benchmark of the B200 partition-method tridiagonal solver (one JSON line).

Workload (BASELINE.json configs[2], the metric's config): one diagonally
dominant FP64 SLAE with N = 8e7 rows per GPU, sub-system size m = 10, all
three stages on the GPU, inputs resident in HBM (2.56 GB per GPU: larger than
the 126 MB L2, so no flush is needed between steps).  A step is one solve.

  value      whole-job unknowns/s, device-resident (CUDA events, max over ranks)
  e2e        the same metric through pm_solve_host_f64 from page-locked host
             buffers: H2D of a,b,c,d and D2H of x inside every timed step
  roofline   the dominant kernel (Stage 3, 40 algorithmic B/unknown) timed
             with CUDA events on its launch stream, vs MEASURED_PEAKS.json
  cpu_baseline  the CPU oracle port of the paper's partition method on the
             host cores (rank 0, N = 1 only)

--gpus N > 1 (under torchrun): one system of N * 8e7 rows row-sharded over
the ranks; the only exchange is the NCCL all-gather of the 64-byte interface
equations per rank (weak scaling).

--impl reference: the reference's CPU implementation of the path.  The
reference ships no solver, so this times the oracle's
restatement of the paper's partition method (oracle/tridiag_oracle.c) on all
host cores; only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FP64 unknowns/s at N=8e7 (HBM GB/s vs peak); e2e time w/ streams vs CPU ref"
BYTES_SOLVE = 40.0   # Stage 3: read a,b,c,d (32 B) + write x (8 B) per unknown
BYTES_REDUCE = 32.0  # Stage 1: read a,b,c,d
BYTES_TOTAL = 72.0   # whole solve (reduced-system traffic ~64/T B, negligible)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="single", choices=["single", "batch"],
                   help="single: config 3/5 (one system, row-sharded for N>1); "
                        "batch: config 4 (--batch systems of --batch-rows, split over the ranks)")
    p.add_argument("--batch", type=int, default=4096)
    p.add_argument("--batch-rows", type=int, default=100_000)
    p.add_argument("--rows-per-gpu", type=float, default=8e7, help="rows per GPU (N)")
    p.add_argument("--precision", default="f64", choices=["f64", "f32"],
                   help="f32: the FP32 solver (pm_*_f32, PAPER.md:243-274); bytes per unknown halve")
    p.add_argument("--m", type=int, default=10)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--num-streams", type=int, default=0, help="e2e stream count (0 = predictor)")
    p.add_argument("--dist-backend", default="nccl", help="torch.distributed backend (tests: gloo)")
    p.add_argument("--exchange", default="auto", choices=["auto", "p2p", "collective"],
                   help="N>1 interface exchange: peer memory (CUDA IPC over NVLink, in-kernel flags) "
                        "or an all-gather; auto = p2p when the mapping self-test passes")
    p.add_argument("--same-device", action="store_true",
                   help="tests only: every rank on cuda:0 (with --dist-backend gloo)")
    p.add_argument("--check", action="store_true",
                   help="gather x on rank 0 and check it against the CPU oracle (small N)")
    p.add_argument("--opt", action="append", default=[],
                   help="solver option NAME=VALUE (PM_OPT_* without the prefix), experiments")
    return p.parse_args()


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            rows = [r.split(",") for r in Path(self.path).read_text().strip().splitlines() if r.strip()]
        except OSError:
            return out
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].lower() == "active":
                    reasons.add(nm)
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(smax), reasons=sorted(reasons),
                       samples=len(sm))
        return out


def cpu_info():
    model = ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def cpu_partition_baseline(n: int, m: int, seed: int, reps: int, warm: int = 1):
    """The oracle port of the paper's partition method, all host threads."""
    import oracle

    a, b, c, d = oracle.generate(n, seed)
    threads = oracle.max_threads()
    times = []
    for k in range(warm + reps):
        t0 = time.perf_counter()
        oracle.partition_solve(a, b, c, d, m, threads)
        dt = time.perf_counter() - t0
        if k >= warm:
            times.append(dt)
    return n / statistics.median(times), threads, times


def cpu_thomas_baseline(n: int, seed: int):
    """Sequential Thomas on one core (SURVEY.md §8d baseline 1), one solve."""
    import oracle

    a, b, c, d = oracle.generate(n, seed)
    t0 = time.perf_counter()
    oracle.thomas(a, b, c, d)
    return n / (time.perf_counter() - t0)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = int(args.rows_per_gpu)
    cores, model = cpu_info()
    ups, threads, times = cpu_partition_baseline(n, args.m, args.seed, args.steps, args.warmup)
    line = {
        "metric": METRIC, "value": ups, "unit": "unknowns/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"single SLAE N={n:.3g} FP64 m={args.m}, CPU partition method "
                               "(Stage 1/3 OpenMP over blocks, serial Stage 2)",
                   "n": n, "m": args.m, "seed": args.seed},
        "cpu_baseline": {"value": ups, "unit": "unknowns/s", "cores": threads, "kind": "port",
                         "sample": f"full N={n} system per step, {args.steps} steps after "
                                   f"{args.warmup} warm-up, median; CPU: {model} ({cores} cpus)"},
        "e2e": {"value": ups, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_batch(args, world, rank, local):
    """BASELINE config 4: `--batch` independent systems of `--batch-rows` rows,
    split contiguously over the ranks with no collective (strong scaling: the
    total batch is fixed).  One step = one pm_solve_batch_device_f64 call on
    this rank's systems (the cluster-per-system kernel: 40 algorithmic B per
    unknown, the Stage-3 re-read served from L2)."""
    import torch
    import torch.distributed as dist

    from paper_2501_05938_b200 import PartitionSolver, pinned_empty
    from paper_2501_05938_b200.solver import PM_OPT_KERNEL_TIMES

    nps, m = args.batch_rows, args.m
    counts = [args.batch // world + (1 if r < args.batch % world else 0) for r in range(world)]
    nb = counts[rank]
    n_loc = nb * nps
    solver = PartitionSolver(local)
    import paper_2501_05938_b200.solver as _solver_mod
    for kv in args.opt:
        name, val = kv.split("=")
        solver.set_option(getattr(_solver_mod, "PM_OPT_" + name.upper()), int(val))
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    first = sum(counts[:rank])
    with torch.cuda.stream(stream):
        # system k of the batch = rows [k*nps, (k+1)*nps) of one long synthetic stream
        a, b, c, d = solver.generate_range_device(args.batch * nps, first * nps, n_loc, args.seed, stream=sh)
        x = torch.empty(n_loc, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()

    def step():
        solver.solve_batch_device(a, b, c, d, n_per_system=nps, m=m, out=x, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    solver.check()
    plan = solver.last_batch_plan()
    launches_per_step = solver.last_launch_count
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    solver.check()
    solver.set_option(PM_OPT_KERNEL_TIMES, 1)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            step()
    torch.cuda.synchronize()
    kt = solver.kernel_times()
    solver.set_option(PM_OPT_KERNEL_TIMES, 0)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    n_total = args.batch * nps
    # e2e: pm_solve_batch_host_f64 from pinned host rows (chunked H2D / solve /
    # D2H on three streams), max over ranks
    e2e = None
    if not args.no_e2e:
        try:
            host = [pinned_empty(n_loc) for _ in range(5)]
        except RuntimeError:
            host = None
        if host is not None:
            for hbuf, t in zip(host, (a, b, c, d)):
                torch.from_numpy(hbuf).copy_(t)
            del a, b, c, d
            torch.cuda.empty_cache()
            solver.solve_batch_host(*host[:4], n_per_system=nps, m=m, out=host[4])  # warm-up
            times = []
            for _ in range(args.e2e_steps):
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                solver.solve_batch_host(*host[:4], n_per_system=nps, m=m, out=host[4])
                times.append(time.perf_counter() - t0)
            t_e2e = statistics.median(times)
            if world > 1:
                t = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                t_e2e = float(t.item())
            e2e = {"value": n_total / t_e2e, "unit": "unknowns/s", "h2d_bytes_per_step": 32 * n_total,
                   "d2h_bytes_per_step": 8 * n_total, "ms_per_step": t_e2e * 1e3,
                   "link_gbs_per_gpu": 40 * n_loc / t_e2e / 1e9, "steps": args.e2e_steps,
                   "timing": "host wall clock around pm_solve_batch_host_f64 (3 streams, chunks of "
                             "~64 MB), median, max over ranks"}
    value = n_total * args.steps / (ms / 1e3)
    peak, peak_src = peaks()
    if plan["cluster"]:
        # one launch per step: the cluster kernel, 40 algorithmic B/unknown
        bpu = 40.0
        kms = sum(t for (md, _, t) in kt if md == 4) / max(1, sum(1 for (md, _, _) in kt if md == 4))
        kname = ("batch_cluster_kernel: 40 B/unknown (a,b,c,d read once from HBM, x written; "
                 "Stage-3 re-read from L2)")
        ach = bpu * n_loc / (kms / 1e3) / 1e9
    else:
        # level kernels over the batch as one long system: dominant kernel =
        # level-0 Stage 3 (40 B/unknown); the whole step moves 72 B/unknown
        bpu = 72.0
        v = [t for (md, lv, t) in kt if md == 1 and lv == 0]
        kms = sum(v) / max(1, len(v))
        kname = "Stage 3 (SOLVE level 0): 40 B/unknown; whole step 72 B/unknown"
        ach = 40.0 * n_loc / (kms / 1e3) / 1e9
    whole = bpu * n_loc / (ms_per_step / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists() and nps == 100_000 and args.batch == 4096 and world == 1:
        try:
            traffic = json.loads(tf.read_text()).get(
                "batch_cluster_bytes_per_launch" if plan["cluster"] else "batch_solve_level0_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based generator, seed %d)" % args.seed,
            "config": {"workload": f"batch of {args.batch} independent FP64 SLAEs, N={nps} each, m={m} "
                                   "(BASELINE config 4), systems split over the ranks",
                       "batch": args.batch, "n_per_system": nps, "m": m, "systems_per_gpu": counts,
                       "parallelism": f"batch-sharded x{world}" if world > 1 else "single GPU",
                       "cluster_plan": plan,
                       "l2": "inputs %.1f GB/GPU > 126 MB L2 (no flush needed)" % (32 * n_loc / 1e9)},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": traffic, "kernel": kname, "peak_source": peak_src, "kernel_ms": kms,
                         "whole_step": {"achieved": whole, "frac": whole / peak, "bytes_per_unknown": bpu}},
            "e2e": e2e,
            "cpu_baseline": None,
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    solver.close()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2501_05938_b200 import PartitionSolver, pinned_empty
    from paper_2501_05938_b200.dist import DistributedSolver, split_rows
    from paper_2501_05938_b200.solver import PM_OPT_KERNEL_TIMES

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)

    if args.workload == "batch":
        return run_batch(args, world, rank, local)
    m = args.m
    rdt = torch.float64 if args.precision == "f64" else torch.float32
    esz = 8 if args.precision == "f64" else 4  # bytes per real
    b_solve, b_reduce, b_total = BYTES_SOLVE * esz / 8, BYTES_REDUCE * esz / 8, BYTES_TOTAL * esz / 8
    n_rank = int(args.rows_per_gpu)
    n_total = n_rank * world
    rows = split_rows(n_total, world, m)
    n_loc = rows[rank]
    row0 = sum(rows[:rank])

    solver = PartitionSolver(local)
    import paper_2501_05938_b200.solver as _solver_mod
    for kv in args.opt:
        name, val = kv.split("=")
        solver.set_option(getattr(_solver_mod, "PM_OPT_" + name.upper()), int(val))
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    with torch.cuda.stream(stream):
        a, b, c, d = solver.generate_range_device(n_total, row0, n_loc, args.seed, stream=sh, dtype=rdt)
        x = torch.empty(n_loc, dtype=rdt, device="cuda")
    torch.cuda.synchronize()
    dsolver = DistributedSolver(solver, exchange=args.exchange) if world > 1 else None

    def step():
        if dsolver is None:
            solver.solve_device(a, b, c, d, m=m, out=x, stream=sh)
        else:
            dsolver.solve(a, b, c, d, x, m=m, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    solver.check()
    launches_per_step = solver.last_launch_count + (1 if world > 1 else 0)

    # ---- timed region: device-resident solves ---------------------------------
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    solver.check()
    # ---- per-kernel CUDA-event times (same steps again, events bracketing every
    # launch on its stream; kept out of the region above because events between
    # launches would serialise the programmatic dependent launches) ----------
    solver.set_option(PM_OPT_KERNEL_TIMES, 1)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            step()
    torch.cuda.synchronize()
    ktimes = solver.kernel_times()
    solver.set_option(PM_OPT_KERNEL_TIMES, 0)
    solver.check()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = n_total * args.steps / (ms / 1e3)

    def gather_check(x_local):
        """Gather the ranks' rows on rank 0 and check them against the oracle."""
        import numpy as np

        xs = x_local.double().cpu()
        if world > 1:
            mx = max(rows)
            buf = torch.zeros(mx, dtype=torch.float64)
            buf[:n_loc] = xs
            parts = [torch.empty(mx, dtype=torch.float64) for _ in range(world)]
            g = dist.new_group(backend="gloo")
            dist.all_gather(parts, buf, group=g)
            xs = torch.cat([p[:k] for p, k in zip(parts, rows)])
        if rank != 0:
            return None
        import oracle

        ah, bh, ch, dh = oracle.generate(n_total, args.seed)
        xr = oracle.thomas(ah, bh, ch, dh)
        xn = np.ascontiguousarray(xs.numpy())
        return {"rel_err": oracle.rel_err(xn, xr), "residual": oracle.residual(ah, bh, ch, dh, xn)}

    check = gather_check(x) if args.check else None

    # dominant kernel: level-0 Stage 3 (mode 1); Stage 1 (mode 0) beside it
    def avg(mode, level=0):
        v = [t for (md, lv, t) in ktimes if md == mode and lv == level]
        return (sum(v) / len(v)) if v else float("nan")

    t_solve, t_reduce = avg(1), avg(0)
    per_kernel = {}
    for (md, lv, t) in ktimes:
        per_kernel.setdefault(f"{['reduce', 'solve', 'root', 'upper', 'cluster'][md]}_L{lv}", []).append(t)
    per_kernel = {k: round(sum(v) / len(v), 5) for k, v in sorted(per_kernel.items())}
    t_kern_total = sum(t for (_, _, t) in ktimes) / args.steps
    peak, peak_src = peaks()
    ach_solve = b_solve * n_loc / (t_solve / 1e3) / 1e9
    ach_reduce = b_reduce * n_loc / (t_reduce / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("solve_level0_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    # ---- e2e through the public host API: pinned host rows in, x out --------
    # N = 1: pm_solve_host_f64 (chunked H2D -> Stage 1 per stream, upper
    # levels, Stage 3 -> D2H per stream; stream count from the predictor).
    # N > 1: DistributedSolver.solve_host on every rank (H2D of the rank's
    # rows, row-sharded solve with the NCCL all-gather, D2H), max over ranks.
    e2e = None
    if not args.no_e2e:
        host = [pinned_empty(n_loc, np.float64 if esz == 8 else np.float32) for _ in range(5)]
        for hbuf, t in zip(host, (a, b, c, d)):
            torch.from_numpy(hbuf).copy_(t)  # the same synthetic rows, staged once
        del a, b, c, d
        torch.cuda.empty_cache()
        xs = host[4]
        ns = args.num_streams
        used = 1
        if world == 1:
            def e2e_step():
                solver.solve_host(*host[:4], m=m, num_streams=ns, out=xs)
        else:
            def e2e_step():
                dsolver.solve_host(*host[:4], xs, m=m, stream=stream)
        for _ in range(2):
            e2e_step()
        times = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_step()
            times.append(time.perf_counter() - t0)
            if world == 1:
                _, _, used = solver.last_stage_timings()
        t_e2e = statistics.median(times)
        if world > 1:
            t = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        e2e = {"value": n_total / t_e2e, "unit": "unknowns/s", "h2d_bytes_per_step": 4 * esz * n_total,
               "d2h_bytes_per_step": esz * n_total, "ms_per_step": t_e2e * 1e3,
               "num_streams": used if world == 1 else None,
               "link_gbs_per_gpu": 5 * esz * n_loc / t_e2e / 1e9, "steps": args.e2e_steps,
               "timing": ("host wall clock around pm_solve_host_%s, median" % args.precision if world == 1 else
                          "host wall clock around DistributedSolver.solve_host per rank, median, max over ranks")}
        if args.check:
            ce = gather_check(torch.from_numpy(xs))
            if check is not None and ce is not None:
                check["e2e"] = ce

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.precision == "f64":
        cores, model = cpu_info()
        ups, threads, times = cpu_partition_baseline(n_loc, m, args.seed, reps=3)
        cpu = {"value": ups, "unit": "unknowns/s", "cores": threads, "kind": "port",
               "sample": f"full N={n_loc} system, median of 3 after 1 warm-up; oracle partition "
                         f"method, Stage 1/3 OpenMP, Stage 2 serial; CPU: {model} ({cores} cpus)",
               "thomas_1core": {"value": cpu_thomas_baseline(n_loc, args.seed), "unit": "unknowns/s",
                                "cores": 1, "sample": f"one sequential Thomas solve of N={n_loc}"}}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (counter-based generator, seed %d)" % args.seed,
            "config": {"workload": "device-resident single SLAE, N=8e7 rows per GPU, %s, m=%d "
                                   "(BASELINE config 3; N>1: one system row-sharded, config 5)"
                                   % ("FP64" if esz == 8 else "FP32 (PAPER.md:243-274 variant)", m),
                       "n_total": n_total, "n_per_gpu": n_rank, "m": m,
                       "parallelism": "row-sharded x%d" % world if world > 1 else "single GPU",
                       "exchange": (dsolver.exchange if dsolver is not None else None),
                       "l2": "inputs %.2f GB/GPU > 126 MB L2 (no flush needed)" % (4 * esz * n_loc / 1e9)},
            "roofline": {"bound": "hbm", "achieved": ach_solve, "peak": peak, "unit": "GB/s",
                         "frac": ach_solve / peak, "traffic": traffic if esz == 8 else None,
                         "kernel": "Stage 3 (SOLVE level 0): %g B/unknown" % b_solve, "peak_source": peak_src,
                         "kernel_ms": t_solve,
                         "stage1": {"achieved": ach_reduce, "frac": ach_reduce / peak,
                                    "kernel_ms": t_reduce, "bytes_per_unknown": b_reduce},
                         "whole_solve": {"achieved": b_total * n_loc / (ms_per_step / 1e3) / 1e9,
                                         "frac": b_total * n_loc / (ms_per_step / 1e3) / 1e9 / peak,
                                         "bytes_per_unknown": b_total,
                                         "kernel_ms_sum": t_kern_total},
                         "kernels_ms": per_kernel},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches_per_step * args.steps,
            **({"check": check} if check is not None else {}),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dsolver.close()
        dist.destroy_process_group()
    solver.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
