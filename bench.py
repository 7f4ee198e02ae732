#!/usr/bin/env python
"""Benchmark of the B200 partition-method tridiagonal solver (one JSON line).

Workloads (BASELINE.json configs):
  single (default)  config 3, the metric's config: one diagonally dominant
                    FP64 SLAE with N = 8e7 rows PER GPU, m = 10, all three
                    stages on the GPU, inputs resident in HBM (2.56 GB per GPU,
                    larger than the 126 MB L2: no flush needed between steps).
                    N GPUs: one system of N * 8e7 rows row-sharded over the
                    ranks (weak scaling).  The line also carries a "c5" object:
                    config 5, one system of N = 1e9 rows split over the same
                    ranks (strong scaling), timed and checked the same way.
  c5                config 5 as the headline line (N = 1e9 total, strong).
  batch             config 4: 4096 independent systems of 1e5 rows, split
                    over the ranks with no collective (strong scaling).

A step is one solve.  Keys:
  value         whole-job unknowns/s, device-resident (CUDA events on the
                launch stream, max over ranks)
  e2e           the same metric through the public host API (pm_solve_host_f64
                / DistributedSolver.solve_host) from page-locked host buffers:
                H2D of a,b,c,d and D2H of x inside every timed step; plus the
                pinned H2D / D2H bandwidth measured in this run and the
                fraction of the link bound 32N/BW_h2d + 8N/BW_d2h achieved
  roofline      the dominant kernel (Stage 3, 40 algorithmic B/unknown),
                CUDA-event time on its launch stream, vs MEASURED_PEAKS.json;
                traffic = ncu DRAM bytes captured for THIS kernel build
                (profiles/ncu_traffic.json, stamped with the source hash)
  exchanges     N > 1: the step time with each interface exchange -- peer
                memory written by the solve kernels themselves (p2p) and the
                NCCL all-gather of the 64-byte interface equations (collective)
  cpu_baseline  the CPU oracle port of the paper's partition method on the
                host cores (rank 0, N = 1 only)

--gpus N > 1 without torchrun: bench.py relaunches itself under
`python -m torch.distributed.run --nproc-per-node N` (exits non-zero when
fewer than N GPUs are visible, unless --same-device).

--impl reference: the reference's CPU implementation of the path.  The
reference ships no solver, so this times the oracle's
restatement of the paper's partition method (oracle/tridiag_oracle.c) on all
host cores on a bounded sample of the same workload; only rank 0 runs it,
and its `config` is the same object this arm prints.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
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
CPU_SAMPLE_ROWS = 80_000_000  # reference arm: bounded sample per step
SELF_LAUNCH_ENV = "PM_BENCH_SELF_LAUNCHED"


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="single", choices=["single", "c5", "batch"],
                   help="single: config 3 (8e7 rows per GPU, row-sharded for N>1; weak) + a c5 object; "
                        "c5: config 5 (1e9 rows total over the ranks; strong); "
                        "batch: config 4 (--batch systems of --batch-rows, split over the ranks)")
    p.add_argument("--batch", type=int, default=4096)
    p.add_argument("--batch-rows", type=int, default=100_000)
    p.add_argument("--rows-per-gpu", type=float, default=8e7, help="rows per GPU of the single workload")
    p.add_argument("--c5-rows", type=float, default=1e9, help="total rows of the c5 workload")
    p.add_argument("--no-c5", action="store_true", help="single workload: skip the c5 object")
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
                   help="N>1 interface exchange of the headline value: peer memory (CUDA IPC over "
                        "NVLink, in-kernel flags) or an all-gather; auto = p2p when the mapping "
                        "self-test passes.  Both are timed and reported under `exchanges`.")
    p.add_argument("--same-device", action="store_true",
                   help="tests only: every rank on cuda:0 (with --dist-backend gloo)")
    p.add_argument("--check", action="store_true",
                   help="check the headline solve against the CPU oracle (windowed Thomas over every "
                        "row, per rank; the c5 object is always checked)")
    p.add_argument("--opt", action="append", default=[],
                   help="solver option NAME=VALUE (PM_OPT_* without the prefix), experiments")
    return p.parse_args(argv)


# ---------------------------------------------------------------------------
# launch plumbing
# ---------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: one process per GPU via torch.distributed.run."""
    if not args.same_device:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"error: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
            return 2
    env = dict(os.environ)
    env[SELF_LAUNCH_ENV] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


SPEC_HBM_GBS = 8000.0  # north_star "about 8 TB/s" (B200_PROFILING.md: 7.7 HGX / 8 DGX)


def kernel_build_hash() -> str:
    """Hash of the solver's CUDA sources: ncu traffic figures are only quoted
    for the build they were captured on."""
    h = hashlib.sha256()
    csrc = ROOT / "paper_2501_05938_b200" / "csrc"
    for p in sorted(list(csrc.glob("*.cu")) + list(csrc.glob("*.cuh")) + list(csrc.glob("*.h")) +
                    list(csrc.glob("*.inc"))):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def traffic_for(key: str):
    """(bytes per launch, provenance) from profiles/ncu_traffic.json when it was
    captured on this kernel build, else (None, why)."""
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if not tf.exists():
        return None, "no capture"
    try:
        doc = json.loads(tf.read_text())
    except (OSError, ValueError):
        return None, "unreadable capture"
    cur = kernel_build_hash()
    if doc.get("build_hash") != cur:
        return None, f"stale: captured on build {doc.get('build_hash')}, running {cur}"
    v = doc.get(key)
    return v, (f"ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, build {cur} "
               f"({doc.get('source', '')})" if v is not None else f"{key} not captured")


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


# ---------------------------------------------------------------------------
# workload description (shared by both arms so the driver sees one config)
# ---------------------------------------------------------------------------
def workload(args, world: int) -> dict:
    prec = "FP64" if args.precision == "f64" else "FP32 (PAPER.md:243-274 variant)"
    if args.workload == "batch":
        n_total = args.batch * args.batch_rows
        return {"workload": f"batch of {args.batch} independent {prec} SLAEs, N={args.batch_rows} each, "
                            f"m={args.m} (BASELINE config 4), systems split over the ranks",
                "batch": args.batch, "n_per_system": args.batch_rows, "n_total": n_total, "m": args.m,
                "seed": args.seed, "precision": args.precision,
                "parallelism": f"batch-sharded x{world}" if world > 1 else "single GPU",
                "scaling": "strong",
                "l2": "inputs %.1f GB/GPU > 126 MB L2 (no flush needed)" % (32 * n_total / world / 1e9)}
    if args.workload == "c5":
        n_total = int(args.c5_rows)
        return {"workload": f"device-resident single {prec} SLAE, N={n_total:.3g} rows in total, m={args.m} "
                            "(BASELINE config 5), row-sharded over the ranks",
                "n_total": n_total, "n_per_gpu": n_total / world, "m": args.m, "seed": args.seed,
                "precision": args.precision,
                "parallelism": f"row-sharded x{world}" if world > 1 else "single GPU",
                "scaling": "strong", "l2": "inputs > 126 MB L2 (no flush needed)"}
    n_rank = int(args.rows_per_gpu)
    esz = 8 if args.precision == "f64" else 4
    return {"workload": f"device-resident single {prec} SLAE, N={n_rank:.3g} rows per GPU, m={args.m} "
                        "(BASELINE config 3; N>1: one system row-sharded over the ranks)",
            "n_total": n_rank * world, "n_per_gpu": n_rank, "m": args.m, "seed": args.seed,
            "precision": args.precision,
            "parallelism": f"row-sharded x{world}" if world > 1 else "single GPU",
            "scaling": "weak",
            "l2": "inputs %.2f GB/GPU > 126 MB L2 (no flush needed)" % (4 * esz * n_rank / 1e9)}


# ---------------------------------------------------------------------------
# reference arm (CPU port of the paper's method; rank 0 only)
# ---------------------------------------------------------------------------
def cpu_partition_baseline(n: int, m: int, seed: int, reps: int, warm: int = 1, batch_rows: int = 0):
    """The oracle port of the paper's partition method, all host threads.
    batch_rows > 0: the rows form independent systems of that size (couplings
    at the system boundaries zeroed), solved in one call."""
    import oracle

    a, b, c, d = oracle.generate(n, seed)
    if batch_rows > 0:
        a[::batch_rows] = 0.0
        c[batch_rows - 1::batch_rows] = 0.0
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
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    cfg = workload(args, world)
    n_total = cfg["n_total"]
    bs = args.batch_rows if args.workload == "batch" else 0
    n = min(n_total, CPU_SAMPLE_ROWS)
    if bs:
        n = max(bs, n // bs * bs)
    cores, model = cpu_info()
    ups, threads, times = cpu_partition_baseline(n, args.m, args.seed, args.steps, args.warmup, batch_rows=bs)
    sample = (f"{'the first %d systems' % (n // bs) if bs else 'a %d-row system' % n} of the same generator "
              f"per step (of the workload's {n_total} rows; unknowns/s is per row), {args.steps} steps "
              f"after {args.warmup} warm-up, median; partition method, Stage 1/3 OpenMP over blocks, "
              f"Stage 2 serial; CPU: {model} ({cores} cpus)")
    line = {
        "metric": METRIC, "value": ups, "unit": "unknowns/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": ups, "unit": "unknowns/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": ups, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class Ctx:
    """Process-group plumbing of one rank."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = 0 if args.same_device else int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.nccl_log = None
        if self.world > 1:
            if args.dist_backend == "nccl":
                # NCCL's own log shows the transport (P2P / NVLS) of the collective exchange
                if "NCCL_DEBUG" not in os.environ:
                    os.environ["NCCL_DEBUG"] = "INFO"
                    os.environ["NCCL_DEBUG_SUBSYS"] = "INIT,COLL"
                    self.nccl_log = os.path.join(tempfile.gettempdir(),
                                                 f"pm_bench_nccl_{os.getpid()}_r{self.rank}.log")
                    os.environ["NCCL_DEBUG_FILE"] = self.nccl_log
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(args.dist_backend)

    @property
    def dev_collectives(self) -> bool:
        return self.world > 1 and self.dist.get_backend() == "nccl"

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        torch = self.torch
        t = torch.tensor([v], dtype=torch.float64, device="cuda" if self.dev_collectives else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, vals) -> list:
        """All-gather a short list of floats; returns [per-rank list]."""
        torch = self.torch
        t = torch.tensor(list(vals), dtype=torch.float64, device="cuda" if self.dev_collectives else "cpu")
        if self.world == 1:
            return [list(vals)]
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        return [p.cpu().tolist() for p in parts]

    def nccl_summary(self):
        if not self.nccl_log or not os.path.exists(self.nccl_log):
            return None
        lines = Path(self.nccl_log).read_text(errors="replace").splitlines()
        pick = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines
                if any(k in ln for k in ("NCCL version", "via P2P", "via NVLS", "NVLS", "nRanks", "CollNet",
                                         "Connected all", "via SHM", "via NET"))]
        via = sorted({w for ln in lines for w in ("P2P/CUMEM", "P2P/IPC", "P2P/direct", "NVLS", "SHM", "NET")
                      if ("via " + w) in ln or (w == "NVLS" and "NVLS multicast support is available" in ln)})
        return {"log_lines": len(lines), "transports": via, "excerpt": pick[:12]}


def set_opts(solver, opts):
    import paper_2501_05938_b200.solver as sm

    for kv in opts:
        name, val = kv.split("=")
        solver.set_option(getattr(sm, "PM_OPT_" + name.upper()), int(val))


def link_bandwidth(nbytes: int = 1 << 30, reps: int = 5) -> dict:
    """Pinned-host <-> device copy bandwidth of this GPU (GB/s, best of reps,
    CUDA events), measured in the same run as the e2e number."""
    import torch

    n = nbytes // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.fill_(1.0)
    dv = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    out = {}
    for name, dst, src in (("h2d_gbs", dv, h), ("d2h_gbs", h, dv)):
        best = 0.0
        with torch.cuda.stream(s):
            for _ in range(reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                dst.copy_(src, non_blocking=True)
                e1.record(s)
                e1.synchronize()
                best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out[name] = best
    del h, dv
    torch.cuda.empty_cache()
    return out


def check_rank(ctx, x_local, n_total: int, row0: int, seed: int) -> dict:
    """Windowed oracle Thomas over every row of this rank's slice (no copy of
    the system is held; bit-identical to whole-system Thomas on these systems,
    tests/test_oracle.py), combined over ranks: rel_err and residual bars."""
    import oracle

    torch = ctx.torch
    xs = x_local.detach().double().cpu().numpy()
    ends = ctx.gather([xs[0], xs[-1]])
    xl = ends[ctx.rank - 1][1] if ctx.rank > 0 else 0.0
    xr = ends[ctx.rank + 1][0] if ctx.rank + 1 < ctx.world else 0.0
    t0 = time.perf_counter()
    r = oracle.check_generated(xs, n_total, row0, seed, xl, xr)
    dt = time.perf_counter() - t0
    parts = ctx.gather([r["max_err"], r["max_ref"], r["rsq"], r["dsq"], dt])
    del xs
    out = oracle.finish_check([{"max_err": p[0], "max_ref": p[1], "rsq": p[2], "dsq": p[3]} for p in parts])
    return {"rel_err": out["rel_err"], "residual": out["residual"], "rows": n_total,
            "method": "windowed oracle Thomas (pad 1024) over every row, each rank its slice, combined",
            "cpu_s_max": max(p[4] for p in parts), "pass": out["rel_err"] <= 1e-10 and out["residual"] <= 1e-12
            if x_local.dtype == torch.float64 else None}


def solve_phase(ctx, args, solver, n_total: int, exchange: str, timed_steps: int, want_e2e: bool,
                want_check: bool, time_both_exchanges: bool, idle_probe: bool = False):
    """Generate this rank's rows of an n_total-row system, time `timed_steps`
    device-resident solves (+ per-kernel event times), optionally the other
    exchange, the oracle check and the e2e solves.  Returns a dict (per rank;
    times already max-reduced over ranks)."""
    import torch

    from paper_2501_05938_b200 import pinned_empty
    from paper_2501_05938_b200.dist import DistributedSolver, split_rows
    from paper_2501_05938_b200.solver import PM_OPT_KERNEL_TIMES

    world, rank, m = ctx.world, ctx.rank, args.m
    rdt = torch.float64 if args.precision == "f64" else torch.float32
    esz = 8 if args.precision == "f64" else 4
    rows = split_rows(n_total, world, m)
    n_loc, row0 = rows[rank], sum(rows[:rank])
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    with torch.cuda.stream(stream):
        a, b, c, d = solver.generate_range_device(n_total, row0, n_loc, args.seed, stream=sh, dtype=rdt)
        x = torch.empty(n_loc, dtype=rdt, device="cuda")
    torch.cuda.synchronize()
    dsolvers = {}
    if world > 1:
        ds = DistributedSolver(solver, exchange=exchange)
        dsolvers[ds.exchange] = ds
        if time_both_exchanges:
            other = "collective" if ds.exchange == "p2p" else "p2p"
            try:
                dsolvers[other] = DistributedSolver(solver, exchange=other)
            except Exception as e:  # p2p mapping unavailable on this group
                dsolvers[other] = e
    main_ex = next(iter(dsolvers)) if dsolvers else None

    def step_fn(ex):
        if ex is None:
            return lambda: solver.solve_device(a, b, c, d, m=m, out=x, stream=sh)
        ds = dsolvers[ex]
        return lambda: ds.solve(a, b, c, d, x, m=m, stream=stream)

    def timed(fn, steps):
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                fn()
        solver.check()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.barrier()
        torch.cuda.synchronize()
        with ClockSampler(ctx.local) as clk:
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(steps):
                    fn()
                e1.record(stream)
            torch.cuda.synchronize()
        ctx.barrier()
        solver.check()
        return ctx.max(e0.elapsed_time(e1)), clk.summary()

    fn = step_fn(main_ex)
    idle_ms = None
    if idle_probe:
        # one solve from an idle GPU (after the warm-up solves and 1 s of
        # idle): B200 holds its burst clocks for ~40-50 ms of back-to-back
        # solves, then its power limit takes ~10 % (tools/power_probe.py)
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                fn()
        torch.cuda.synchronize()
        time.sleep(1.0)
        ctx.barrier()
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            i0.record(stream)
            fn()
            i1.record(stream)
        torch.cuda.synchronize()
        idle_ms = ctx.max(i0.elapsed_time(i1))
    ms, clocks = timed(fn, timed_steps)
    launches = (dsolvers[main_ex].last_launches if main_ex else solver.last_launch_count)
    # per-kernel CUDA-event times (same steps again, events bracketing every
    # launch on its stream; kept out of the region above because events
    # between launches would serialise the programmatic dependent launches)
    solver.set_option(PM_OPT_KERNEL_TIMES, 1)
    with torch.cuda.stream(stream):
        for _ in range(timed_steps):
            fn()
    torch.cuda.synchronize()
    ktimes = solver.kernel_times()
    solver.set_option(PM_OPT_KERNEL_TIMES, 0)
    solver.check()
    out = {"ms": ms, "ms_per_step": ms / timed_steps, "clocks": clocks, "ktimes": ktimes, "idle_ms": idle_ms,
           "launches_per_step": launches, "n_loc": n_loc, "row0": row0, "rows": rows, "exchange": main_ex}
    if world > 1:
        ex = {main_ex: {"ms_per_step": ms / timed_steps, "value": n_total * timed_steps / (ms / 1e3)}}
        for name, ds in dsolvers.items():
            if name == main_ex:
                continue
            if isinstance(ds, Exception):
                ex[name] = {"unavailable": str(ds)[:200]}
                continue
            ms2, _ = timed(step_fn(name), timed_steps)
            ex[name] = {"ms_per_step": ms2 / timed_steps, "value": n_total * timed_steps / (ms2 / 1e3)}
        out["exchanges"] = ex
    if want_check:  # x holds the last timed solve's result
        out["check"] = check_rank(ctx, x, n_total, row0, args.seed)

    if want_e2e:
        # e2e through the public host API: pinned host rows in, x out.
        # N = 1: pm_solve_host_f64 (chunked H2D -> Stage 1 per stream, upper
        # levels, Stage 3 -> D2H per stream; stream count from the predictor).
        # N > 1: DistributedSolver.solve_host on every rank, max over ranks.
        host = [pinned_empty(n_loc, np.float64 if esz == 8 else np.float32) for _ in range(5)]
        for hbuf, t in zip(host, (a, b, c, d)):
            torch.from_numpy(hbuf).copy_(t)  # the same synthetic rows, staged once
        del a, b, c, d
        torch.cuda.empty_cache()
        xs = host[4]
        used = 1
        if world == 1:
            def e2e_step():
                solver.solve_host(*host[:4], m=m, num_streams=args.num_streams, out=xs)
        else:
            dse = dsolvers[main_ex]

            def e2e_step():
                dse.solve_host(*host[:4], xs, m=m, stream=stream)
        for _ in range(2):
            e2e_step()
        times = []
        for _ in range(args.e2e_steps):
            ctx.barrier()
            t0 = time.perf_counter()
            e2e_step()
            times.append(time.perf_counter() - t0)
            if world == 1:
                _, _, used = solver.last_stage_timings()
        t_e2e = ctx.max(statistics.median(times))
        bw = link_bandwidth()
        bound = (4 * esz * n_loc / (bw["h2d_gbs"] * 1e9) + esz * n_loc / (bw["d2h_gbs"] * 1e9))
        e2e = {"value": n_total / t_e2e, "unit": "unknowns/s", "h2d_bytes_per_step": 4 * esz * n_total,
               "d2h_bytes_per_step": esz * n_total, "ms_per_step": t_e2e * 1e3,
               "num_streams": used if world == 1 else None,
               "link_gbs_per_gpu": 5 * esz * n_loc / t_e2e / 1e9,
               "link_measured": {k: round(v, 2) for k, v in bw.items()},
               "link_bound_ms": bound * 1e3,
               "link_frac": bound / t_e2e,
               "link_frac_note": "(4*esz*N/BW_h2d + esz*N/BW_d2h) / t_e2e per GPU: one system's H2D must "
                                 "finish before any x exists, so the two transfers cannot overlap each other",
               "steps": args.e2e_steps,
               "timing": ("host wall clock around pm_solve_host_%s, median" % args.precision if world == 1 else
                          "host wall clock around DistributedSolver.solve_host per rank, median, max over ranks")}
        if want_check:
            e2e["check"] = check_rank(ctx, torch.from_numpy(xs), n_total, row0, args.seed)
        out["e2e"] = e2e
        del host
    else:
        del a, b, c, d
    del x
    for ds in dsolvers.values():
        if not isinstance(ds, Exception):
            ds.close()
    torch.cuda.empty_cache()
    return out


def roofline(res, esz: int):
    """Dominant kernel = level-0 Stage 3 (mode 1); Stage 1 (mode 0) beside it."""
    kt = res["ktimes"]
    n_loc = res["n_loc"]
    b_solve, b_reduce, b_total = BYTES_SOLVE * esz / 8, BYTES_REDUCE * esz / 8, BYTES_TOTAL * esz / 8

    def avg(mode, level=0):
        v = [t for (md, lv, t) in kt if md == mode and lv == level]
        return (sum(v) / len(v)) if v else float("nan")

    t_solve, t_reduce = avg(1), avg(0)
    per_kernel = {}
    for (md, lv, t) in kt:
        per_kernel.setdefault(f"{['reduce', 'solve', 'root', 'upper', 'cluster'][md]}_L{lv}", []).append(t)
    steps = max(1, sum(1 for (md, lv, _) in kt if md == 1 and lv == 0))
    per_kernel = {k: round(sum(v) / len(v), 5) for k, v in sorted(per_kernel.items())}
    peak, peak_src = peaks()
    ach_solve = b_solve * n_loc / (t_solve / 1e3) / 1e9
    ach_reduce = b_reduce * n_loc / (t_reduce / 1e3) / 1e9
    whole = b_total * n_loc / (res["ms_per_step"] / 1e3) / 1e9
    if n_loc == 80_000_000:
        traffic, tprov = traffic_for("solve_level0_bytes_per_launch" if esz == 8 else "solve_level0_f32_bytes_per_launch")
    else:
        traffic, tprov = None, "captured for the N=8e7 launches (FP64, FP32) only"
    return {"bound": "hbm", "achieved": ach_solve, "peak": peak, "unit": "GB/s", "frac": ach_solve / peak,
            "traffic": traffic, "traffic_source": tprov,
            "kernel": "Stage 3 (SOLVE level 0): %g B/unknown x %d rows per launch" % (b_solve, n_loc),
            "peak_source": peak_src, "kernel_ms": t_solve,
            "stage1": {"achieved": ach_reduce, "frac": ach_reduce / peak, "kernel_ms": t_reduce,
                       "bytes_per_unknown": b_reduce},
            "whole_solve": {"achieved": whole, "frac": whole / peak, "bytes_per_unknown": b_total,
                            "kernel_ms_sum": sum(t for (_, _, t) in kt) / steps,
                            "frac_of_spec": whole / SPEC_HBM_GBS},
            "spec": {"hbm_gbs": SPEC_HBM_GBS, "frac": ach_solve / SPEC_HBM_GBS,
                     "note": "north_star's ~8 TB/s (B200 DGX figure; HGX 7.7 TB/s); frac/peak use the "
                             "measured copy bandwidth"},
            "kernels_ms": per_kernel}


def run_batch(args, ctx):
    """BASELINE config 4: `--batch` independent systems of `--batch-rows` rows,
    split contiguously over the ranks with no collective (strong scaling: the
    total batch is fixed).  One step = one pm_solve_batch_device_f64 call on
    this rank's systems."""
    import torch

    from paper_2501_05938_b200 import PartitionSolver, pinned_empty
    from paper_2501_05938_b200.solver import PM_OPT_KERNEL_TIMES

    world, rank, local = ctx.world, ctx.rank, ctx.local
    nps, m = args.batch_rows, args.m
    counts = [args.batch // world + (1 if r < args.batch % world else 0) for r in range(world)]
    nb = counts[rank]
    n_loc = nb * nps
    solver = PartitionSolver(local)
    set_opts(solver, args.opt)
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
    ctx.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
        torch.cuda.synchronize()
    ctx.barrier()
    ms = ev0.elapsed_time(ev1)
    solver.check()
    solver.set_option(PM_OPT_KERNEL_TIMES, 1)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            step()
    torch.cuda.synchronize()
    kt = solver.kernel_times()
    solver.set_option(PM_OPT_KERNEL_TIMES, 0)
    ms = ctx.max(ms)
    ms_per_step = ms / args.steps
    n_total = args.batch * nps
    check = None
    if args.check:
        # every system's rows checked against oracle Thomas of that system
        import oracle

        xs = x.double().cpu().numpy()
        parts = []
        for k in range(nb):
            lo = (first + k) * nps
            parts.append(_check_batch_system(oracle, xs[k * nps:(k + 1) * nps], args.batch * nps, lo, nps,
                                             args.seed))
        r = oracle.finish_check(parts)
        g = ctx.gather([r["max_err"], r["max_ref"], r["rsq"], r["dsq"]])
        r = oracle.finish_check([{"max_err": p[0], "max_ref": p[1], "rsq": p[2], "dsq": p[3]} for p in g])
        check = {"rel_err": r["rel_err"], "residual": r["residual"], "systems": args.batch}
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
                ctx.barrier()
                t0 = time.perf_counter()
                solver.solve_batch_host(*host[:4], n_per_system=nps, m=m, out=host[4])
                times.append(time.perf_counter() - t0)
            t_e2e = ctx.max(statistics.median(times))
            bw = link_bandwidth()
            # batches pipeline chunks: copy-in of one overlaps copy-out of another
            bound = max(32 * n_loc / (bw["h2d_gbs"] * 1e9), 8 * n_loc / (bw["d2h_gbs"] * 1e9))
            e2e = {"value": n_total / t_e2e, "unit": "unknowns/s", "h2d_bytes_per_step": 32 * n_total,
                   "d2h_bytes_per_step": 8 * n_total, "ms_per_step": t_e2e * 1e3,
                   "link_gbs_per_gpu": 40 * n_loc / t_e2e / 1e9,
                   "link_measured": {k: round(v, 2) for k, v in bw.items()},
                   "link_bound_ms": bound * 1e3, "link_frac": bound / t_e2e,
                   "link_frac_note": "max(32N/BW_h2d, 8N/BW_d2h) / t_e2e per GPU (chunks overlap copy-in "
                                     "with copy-out)",
                   "steps": args.e2e_steps,
                   "timing": "host wall clock around pm_solve_batch_host_f64 (3 streams, chunks of "
                             "~256 MB), median, max over ranks"}
    value = n_total * args.steps / (ms / 1e3)
    peak, peak_src = peaks()
    if plan["kernel"] in ("cluster", "stream"):
        bpu = 40.0
        v = [t for (md, _, t) in kt if md == 4]
        kms = sum(v) / max(1, len(v))
        kname = (f"batch_{plan['kernel']}_kernel: 40 B/unknown (a,b,c,d read once from HBM, x written; "
                 "Stage-3 re-read from L2)")
        ach = bpu * n_loc / (kms / 1e3) / 1e9
        tkey = f"batch_{plan['kernel']}_bytes_per_launch"
    else:
        bpu = 72.0
        v = [t for (md, lv, t) in kt if md == 1 and lv == 0]
        kms = sum(v) / max(1, len(v))
        kname = "Stage 3 (SOLVE level 0): 40 B/unknown; whole step 72 B/unknown"
        ach = 40.0 * n_loc / (kms / 1e3) / 1e9
        tkey = "batch_solve_level0_bytes_per_launch"
    whole = bpu * n_loc / (ms_per_step / 1e3) / 1e9
    traffic, tprov = (traffic_for(tkey) if (nps == 100_000 and args.batch == 4096 and world == 1)
                      else (None, "captured for the 4096 x 1e5 single-GPU launch only"))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based generator, seed %d)" % args.seed,
            "config": workload(args, world),
            "systems_per_gpu": counts, "cluster_plan": plan,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": traffic, "traffic_source": tprov, "kernel": kname, "peak_source": peak_src,
                         "kernel_ms": kms,
                         "whole_step": {"achieved": whole, "frac": whole / peak, "bytes_per_unknown": bpu,
                                        "compulsory_frac": 40.0 * n_loc / (ms_per_step / 1e3) / 1e9 / peak}},
            "e2e": e2e,
            "cpu_baseline": None,
            "gpu_launches": args.steps * launches_per_step,
            **({"check": check} if check is not None else {}),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    solver.close()
    return 0


def _check_batch_system(oracle, xk, n_all: int, lo: int, nps: int, seed: int) -> dict:
    """Oracle Thomas of one batch system (its first a / last c ignored)."""
    a, b, c, d = oracle.generate_range(n_all, lo, nps, seed)
    a[0] = 0.0
    c[-1] = 0.0
    xr = oracle.thomas(a, b, c, d)
    xk = np.ascontiguousarray(xk)
    r = b * xk - d
    r[1:] += a[1:] * xk[:-1]
    r[:-1] += c[:-1] * xk[1:]
    return {"max_err": float(np.max(np.abs(xk - xr))), "max_ref": float(np.max(np.abs(xr))),
            "rsq": float(r @ r), "dsq": float(d @ d)}


def run_single(args, ctx):
    import torch

    from paper_2501_05938_b200 import PartitionSolver

    world, rank = ctx.world, ctx.rank
    esz = 8 if args.precision == "f64" else 4
    cfg = workload(args, world)
    solver = PartitionSolver(ctx.local)
    set_opts(solver, args.opt)
    is_c5 = args.workload == "c5"
    res = solve_phase(ctx, args, solver, cfg["n_total"], args.exchange, args.steps,
                      want_e2e=not args.no_e2e and not is_c5, want_check=args.check or is_c5,
                      time_both_exchanges=True)
    c5 = None
    if not is_c5 and not args.no_c5 and args.precision == "f64":
        # config 5 beside the metric line: 1e9 rows over the same ranks
        n5 = int(args.c5_rows)
        r5 = solve_phase(ctx, args, solver, n5, args.exchange, args.steps, want_e2e=False, want_check=True,
                         time_both_exchanges=True, idle_probe=True)
        rf5 = roofline(r5, esz)
        c5 = {"workload": f"one FP64 SLAE, N={n5:.3g} rows in total, m={args.m} (BASELINE config 5), "
                          f"row-sharded over {world} rank(s) (strong scaling)",
              "n_total": n5, "rows_per_rank": r5["rows"], "value": n5 * args.steps / (r5["ms"] / 1e3),
              "unit": "unknowns/s", "ms_per_step": r5["ms_per_step"], "exchange": r5["exchange"],
              **({"exchanges": r5["exchanges"]} if "exchanges" in r5 else {}),
              "whole_solve_frac": rf5["whole_solve"]["frac"], "stage3_frac": rf5["frac"],
              "stage1_frac": rf5["stage1"]["frac"], "kernels_ms": rf5["kernels_ms"],
              "gpu_launches_per_step": r5["launches_per_step"], "check": r5["check"], "clocks": r5["clocks"],
              "idle_solve": {"ms": r5["idle_ms"],
                             "whole_solve_frac": rf5["whole_solve"]["bytes_per_unknown"] * n5 / max(1, world)
                             / (r5["idle_ms"] / 1e3) / 1e9 / rf5["peak"] if r5["idle_ms"] else None,
                             "note": "one solve after 1 s idle (burst clocks); the timed steps run back to back "
                                     "for ~0.3 s, under the power limit (sw_power_cap)"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.precision == "f64":
        cores, model = cpu_info()
        n_cpu = min(res["n_loc"], CPU_SAMPLE_ROWS)
        ups, threads, times = cpu_partition_baseline(n_cpu, args.m, args.seed, reps=3)
        cpu = {"value": ups, "unit": "unknowns/s", "cores": threads, "kind": "port",
               "sample": f"N={n_cpu} system, median of 3 after 1 warm-up; oracle partition "
                         f"method, Stage 1/3 OpenMP, Stage 2 serial; CPU: {model} ({cores} cpus)",
               "thomas_1core": {"value": cpu_thomas_baseline(n_cpu, args.seed), "unit": "unknowns/s",
                                "cores": 1, "sample": f"one sequential Thomas solve of N={n_cpu}"}}

    nccl = ctx.nccl_summary()
    if rank == 0:
        n_total = cfg["n_total"]
        line = {
            "metric": METRIC, "value": n_total * args.steps / (res["ms"] / 1e3), "unit": "unknowns/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (counter-based generator, seed %d)" % args.seed,
            "config": cfg,
            "exchange": res["exchange"],
            **({"exchanges": res["exchanges"]} if "exchanges" in res else {}),
            "roofline": roofline(res, esz),
            "e2e": res.get("e2e"),
            "cpu_baseline": cpu,
            "gpu_launches": res["launches_per_step"] * args.steps,
            **({"check": res["check"]} if "check" in res else {}),
            **({"c5": c5} if c5 is not None else {}),
            **({"nccl": nccl} if nccl is not None else {}),
            "clocks": res["clocks"],
        }
        print(json.dumps(line), flush=True)
    solver.close()
    return 0


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "ours" and args.gpus > 1 and env_world is None:
        return self_launch(args)
    if env_world is not None and int(env_world) != args.gpus:
        print(f"error: --gpus {args.gpus} but WORLD_SIZE {env_world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and args.dist_backend == "nccl" and not args.same_device:
        import torch

        if torch.cuda.device_count() < args.gpus:
            print(f"error: --gpus {args.gpus} needs {args.gpus} visible GPUs, found "
                  f"{torch.cuda.device_count()}", file=sys.stderr)
            return 2
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and "OMP_NUM_THREADS" not in os.environ:
        # the per-rank oracle checks share the host's cores
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // int(os.environ["WORLD_SIZE"])))
    ctx = Ctx(args)
    try:
        if args.workload == "batch":
            return run_batch(args, ctx)
        return run_single(args, ctx)
    finally:
        if ctx.world > 1:
            ctx.dist.barrier()
            ctx.dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
