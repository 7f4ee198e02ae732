#!/usr/bin/env python
"""B200 re-fit of the paper's stream-count models (BASELINE.json config 2).

The C2 sweep: 30 SLAE sizes {1, 2.5, 4, 5, 7.5, 8} x 10^i, i = 3..7, m = 10,
num_streams in {1, 2, 4, 8, 16, 32}, end to end through pm_solve_host_f64
from page-locked host buffers (PAPER.md:52 sizes; PAPER.md:60 counts).

1. StageTimings per size, measured unstreamed with CUDA events
   (PM_OPT_TIMINGS; t1_d2h = t3_h2d = 0 because the reduced system never
   leaves the device, t2_comp = the GPU reduced solve).
2. T_str per (size, n): median of `reps` solves (the handle's event total).
3. The two CSV documents of SPEC.md:349/359 are written and fed to the C++
   fit (st_fit_bundle = cmd_fit: Eq. 4 sum model, Eq. 7
   small/big overhead models, 3:1 split, seed 42).
4. Validation: for every size, the bundle's recommend() vs the measured
   optimum; the north_star bar is "within one power of two".

Outputs (default --out refit/): stage_timings.csv, streamed_runs.csv,
bundle.json (SPEC.md:316 keys), validation.json; --install also writes
paper_2501_05938_b200/csrc/streamtune/b200_bundle.inc, the compiled-in
default of the C ABI's predictor.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2501_05938_b200 import PartitionSolver, pinned_empty  # noqa: E402
from paper_2501_05938_b200 import streamtune as st  # noqa: E402
from paper_2501_05938_b200.solver import PM_OPT_STREAM_MODE, PM_OPT_TIMINGS  # noqa: E402

SIZES = [int(k * 10**i) for i in range(3, 8) for k in (1, 2.5, 4, 5, 7.5, 8)]
COUNTS = [1, 2, 4, 8, 16, 32]


def synthetic(n: int, seed: int = 42, precision: str = "f64"):
    """The counter-based system, generated on the device and copied to pinned
    host buffers (the same bits as the CPU oracle's generator; FP32: their
    round-to-nearest images)."""
    import numpy as np
    import torch

    dt = torch.float64 if precision == "f64" else torch.float32
    s = PartitionSolver(0)
    arrs = s.generate_device(n, seed, dtype=dt)
    torch.cuda.synchronize()
    host = []
    for t in arrs:
        h = pinned_empty(n, np.float64 if precision == "f64" else np.float32)
        h[:] = t.cpu().numpy()
        host.append(h)
    s.close()
    del arrs
    return host


def sweep(sizes, reps: int, stream_mode: int, m: int = 10, precision: str = "f64"):
    solver = PartitionSolver(0)
    solver.set_option(PM_OPT_STREAM_MODE, stream_mode)
    stage_rows, run_rows, raw = [], [], {}
    for n in sizes:
        a, b, c, d = synthetic(n, precision=precision)
        x = pinned_empty(n, b.dtype)
        # warm-up every count once (stream pools, allocations)
        for ns in COUNTS:
            solver.solve_host(a, b, c, d, m=m, num_streams=ns, out=x)
        # StageTimings, unstreamed
        solver.set_option(PM_OPT_TIMINGS, 1)
        comps = []
        for _ in range(reps):
            solver.solve_host(a, b, c, d, m=m, num_streams=1, out=x)
            comps.append(solver.last_stage_timings()[0])
        solver.set_option(PM_OPT_TIMINGS, 0)
        med = {f: statistics.median(getattr(t, f) for t in comps)
               for f in ("t1_h2d", "t1_comp", "t1_d2h", "t2_comp", "t3_h2d", "t3_comp", "t3_d2h")}
        stage_rows.append((n, med))
        # T_str per count, interleaved repetitions
        times = {ns: [] for ns in COUNTS}
        for _ in range(reps):
            for ns in COUNTS:
                solver.solve_host(a, b, c, d, m=m, num_streams=ns, out=x)
                times[ns].append(solver.last_stage_timings()[1])
        for ns in COUNTS:
            run_rows.append((n, ns, statistics.median(times[ns])))
        raw[n] = {str(k): v for k, v in times.items()}
        best = min(COUNTS, key=lambda k: statistics.median(times[k]))
        print(f"N={n:>9d}  T_non_str={statistics.median(times[1]):9.4f} ms  "
              f"best n={best:2d} ({statistics.median(times[best]):9.4f} ms)  "
              f"components={ {k: round(v, 4) for k, v in med.items()} }", flush=True)
        del a, b, c, d, x
    solver.close()
    return stage_rows, run_rows, raw


def to_csv(stage_rows, run_rows):
    s = "slae_size,t1_h2d,t1_comp,t1_d2h,t2_comp,t3_h2d,t3_comp,t3_d2h\n"
    for n, t in stage_rows:
        s += f"{n},{t['t1_h2d']!r},{t['t1_comp']!r},{t['t1_d2h']!r},{t['t2_comp']!r},{t['t3_h2d']!r}," \
             f"{t['t3_comp']!r},{t['t3_d2h']!r}\n"
    r = "slae_size,num_streams,t_str\n"
    for n, ns, t in run_rows:
        r += f"{n},{ns},{t!r}\n"
    return s, r


def tie_set(times: dict, z: float = 2.0) -> list[int]:
    """Stream counts whose median time is statistically indistinguishable from
    the best one: median(k) - median(best) <= z * sqrt(se_k^2 + se_best^2),
    se = 1.2533 * 1.4826 * MAD / sqrt(reps) (standard error of a median)."""
    def med_se(v):
        md = statistics.median(v)
        mad = statistics.median(abs(x - md) for x in v)
        return md, 1.2533 * 1.4826 * mad / math.sqrt(max(1, len(v)))
    ms = {k: med_se(v) for k, v in times.items()}
    best = min(ms, key=lambda k: ms[k][0])
    return sorted(k for k in ms
                  if ms[k][0] - ms[best][0] <= z * math.sqrt(ms[k][1] ** 2 + ms[best][1] ** 2))


def validate(bundle, run_rows, raw=None):
    """Predicted vs measured optimum per size.  Strict: the argmin of the
    medians.  Tie-aware (when the per-repetition times are available): the
    measured optimum is the set of counts within measurement noise of the
    best (tie_set), since on B200 most curves are flat to < 1 %."""
    by = {}
    for n, ns, t in run_rows:
        by.setdefault(n, {})[ns] = t
    out = []
    for n in sorted(by):
        meas = min(by[n], key=lambda k: by[n][k])
        pred = st.recommend(bundle, n).chosen
        ratio = max(pred, meas) / min(pred, meas)
        row = {"slae_size": n, "measured_opt": meas, "predicted": pred,
               "within_one_power_of_two": ratio <= 2,
               "t_pred_over_t_best": by[n][pred] / by[n][meas]}
        rk = raw.get(n, raw.get(str(n))) if raw else None
        if rk:
            ties = tie_set({int(k): v for k, v in rk.items()})
            row.update(measured_ties=ties, predicted_in_ties=pred in ties,
                       within_one_power_of_two_of_ties=any(max(pred, k) / min(pred, k) <= 2 for k in ties))
        out.append(row)
    return out


def summarize(val, met):
    s = {"sizes": len(val), "exact": sum(v["predicted"] == v["measured_opt"] for v in val),
         "within_one_power_of_two": sum(v["within_one_power_of_two"] for v in val),
         "worst_t_pred_over_t_best": max(v["t_pred_over_t_best"] for v in val), "metrics": met}
    if all("measured_ties" in v for v in val):
        s["tie_aware"] = {"exact": sum(v["predicted_in_ties"] for v in val),
                          "within_one_power_of_two": sum(v["within_one_power_of_two_of_ties"] for v in val),
                          "rule": "measured optimum = counts within 2 standard errors of the best median"}
    s["rows"] = val
    return s


def validate_fp32(bundle64, bundle32, run_rows):
    """Table 5 on B200: the measured FP32 optimum against the paper's halving
    rule applied to the FP64 bundle (recommend_fp32) and against
    the FP32 re-fit's own recommendation."""
    by = {}
    for n, ns, t in run_rows:
        by.setdefault(n, {})[ns] = t
    out = []
    for n in sorted(by):
        meas = min(by[n], key=lambda k: by[n][k])
        half = st.recommend_fp32(bundle64, n)
        fit = st.recommend(bundle32, n).chosen
        out.append({"slae_size": n, "measured_opt_fp32": meas, "fp64_choice": st.recommend(bundle64, n).chosen,
                    "halving_rule": half, "fp32_fit": fit,
                    "halving_within_one_power_of_two": max(half, meas) / min(half, meas) <= 2,
                    "fit_within_one_power_of_two": max(fit, meas) / min(fit, meas) <= 2,
                    "t_half_over_t_best": by[n][half] / by[n][meas],
                    "t_fit_over_t_best": by[n][fit] / by[n][meas]})
    return out


def write_inc(bundle, path: Path, note: str):
    path.write_text(
        "// Generated by tools/refit.py -- the B200 re-fit of the paper's Eq. 4 / Eq. 7\n"
        f"// ({note}).  Used by streamtune::ModelBundle::b200().\n"
        f"b.sum_a = {bundle.sum_a!r};\nb.sum_b = {bundle.sum_b!r};\n"
        f"b.small_a = {bundle.small_a!r};\nb.small_b = {bundle.small_b!r};\nb.small_c = {bundle.small_c!r};\n"
        f"b.big_a = {bundle.big_a!r};\nb.big_b = {bundle.big_b!r};\nb.big_c = {bundle.big_c!r};\n"
        f"b.size_threshold = {int(bundle.size_threshold)};\n")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--out", default="refit")
    p.add_argument("--stream-mode", type=int, default=0, help="0 pooled streams, 1 created per solve")
    p.add_argument("--max-size", type=float, default=8e7)
    p.add_argument("--threshold", type=int, default=1_000_000)
    p.add_argument("--install", action="store_true")
    p.add_argument("--precision", default="f64", choices=["f64", "f32"],
                   help="f32: the FP32 sweep (pm_solve_host_f32) and Table 5 on B200")
    p.add_argument("--overhead-fit", default="anchored", choices=["anchored", "ols"],
                   help="anchored: T_overhead(N, 1) = 0 and coefficients >= 0 (the B200 default); "
                        "ols: the SPEC's unconstrained least squares")
    p.add_argument("--from-dir", default=None,
                   help="refit from the CSVs (+ raw_times.json) of an earlier sweep in this directory "
                        "instead of measuring (no GPU)")
    args = p.parse_args()
    out = ROOT / args.out
    out.mkdir(parents=True, exist_ok=True)
    t0 = time.time()
    if args.from_dir:
        src = ROOT / args.from_dir
        stage_csv = (src / "stage_timings.csv").read_text()
        runs_csv = (src / "streamed_runs.csv").read_text()
        raw = json.loads((src / "raw_times.json").read_text()) if (src / "raw_times.json").exists() else None
        run_rows = st.load_streamed_runs(runs_csv)
        prev = json.loads((src / "bundle.json").read_text()).get("provenance", {}) if (src / "bundle.json").exists() \
            else {}
        sweep_info = {k: prev[k] for k in ("stream_mode", "reps", "sweep_seconds") if k in prev}
    else:
        sizes = [n for n in SIZES if n <= args.max_size]
        stage_rows, run_rows, raw = sweep(sizes, args.reps, args.stream_mode, precision=args.precision)
        stage_csv, runs_csv = to_csv(stage_rows, run_rows)
        (out / "stage_timings.csv").write_text(stage_csv)
        (out / "streamed_runs.csv").write_text(runs_csv)
        (out / "raw_times.json").write_text(json.dumps(raw))
        sweep_info = {"stream_mode": "pooled" if args.stream_mode == 0 else "created per solve",
                      "reps": args.reps, "sweep_seconds": round(time.time() - t0, 1)}
    bundle, met = st.fit_bundle(stage_csv, runs_csv, size_threshold=args.threshold, seed=42,
                                anchored=args.overhead_fit == "anchored")
    bundle.provenance.update({"fitted_on": f"NVIDIA B200 (tools/refit.py, pm_solve_host_{args.precision}, m=10)",
                              "overhead_fit": args.overhead_fit, **sweep_info})
    (out / "bundle.json").write_text(json.dumps(bundle.to_document(), indent=1))
    val = validate(bundle, run_rows, raw)
    summary = summarize(val, met)
    if args.precision == "f32":
        t5 = validate_fp32(st.ModelBundle.b200(), bundle, run_rows)
        summary["table5_b200"] = {
            "halving_exact": sum(r["halving_rule"] == r["measured_opt_fp32"] for r in t5),
            "halving_within_one_power_of_two": sum(r["halving_within_one_power_of_two"] for r in t5),
            "fp32_fit_exact": sum(r["fp32_fit"] == r["measured_opt_fp32"] for r in t5),
            "fp32_fit_within_one_power_of_two": sum(r["fit_within_one_power_of_two"] for r in t5),
            "worst_t_half_over_t_best": max(r["t_half_over_t_best"] for r in t5),
            "rows": t5}
    (out / "validation.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: (v if k != "table5_b200" else {kk: vv for kk, vv in v.items() if kk != "rows"})
                      for k, v in summary.items() if k != "rows"}, indent=1))
    if args.install and args.precision == "f64":
        write_inc(bundle, ROOT / "paper_2501_05938_b200" / "csrc" / "streamtune" / "b200_bundle.inc",
                  f"{len(val)} sizes x {len(COUNTS)} stream counts, {sweep_info.get('reps')} reps, "
                  f"{sweep_info.get('stream_mode')} streams, {args.overhead_fit} overhead fit")


if __name__ == "__main__":
    main()
