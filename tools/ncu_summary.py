#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list (--csv --log-file of
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`)
and `--set full` reports (.ncu-rep, read with `ncu -i ... --page raw --csv`).

  python tools/ncu_summary.py launches LIST.csv [--step-kernels K] [--bytes name=B ...]
  python tools/ncu_summary.py full REPORT.ncu-rep [...]

Prints markdown.  ncu times are cold-cache and serialised: compare shares,
not absolute times (the bench's live CUDA-event times are the numbers).
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess
import sys
from collections import OrderedDict

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def _val(v: str, unit: str) -> float:
    v = v.replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return float("nan")
    return x * UNITS.get(unit, 1.0)


def launches(path: str, last: int, algo: dict) -> str:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = OrderedDict()
    for r in rows:
        k = (r["ID"], r["Kernel Name"])
        per.setdefault(k, {})[r["Metric Name"]] = _val(r["Metric Value"], r["Metric Unit"])
    items = list(per.items())
    if last:
        items = items[-last:]
    total = sum(m.get("gpu__time_duration.sum", 0.0) for _, m in items)
    out = ["| id | kernel | ncu time (us) | share | DRAM read (GB) | DRAM write (GB) | algorithmic (GB) | traffic / algorithmic |",
           "|---|---|---|---|---|---|---|---|"]
    for (i, name), m in items:
        t = m.get("gpu__time_duration.sum", 0.0)
        rd = m.get("dram__bytes_read.sum", 0.0) / 1e9
        wr = m.get("dram__bytes_write.sum", 0.0) / 1e9
        short = name.split("(")[0]
        a = next((v for k, v in algo.items() if k in name), None)
        ratio = f"{(rd + wr) / a:.3f}" if a else "-"
        out.append(f"| {i} | `{short}` | {t:.1f} | {100 * t / total:.1f}% | {rd:.3f} | {wr:.3f} | "
                   f"{a if a else '-'} | {ratio} |")
    out.append(f"\nTotal of the listed launches under ncu: {total:.1f} us.")
    return "\n".join(out)


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__cluster_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full(path: str) -> str:
    res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True)
    rows = list(csv.reader(io.StringIO(res.stdout)))
    head, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        kv = dict(zip(head, d))
        un = dict(zip(head, units))
        out.append(f"### `{kv.get('Kernel Name', '?').split('(')[0]}` (id {kv.get('ID', '?')})\n")
        out.append("| metric | value |\n|---|---|")
        for k in FULL:
            if k in kv:
                out.append(f"| {k} | {kv[k]} {un.get(k, '')} |")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): _val(v, "")
                  for k, v in kv.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(v for v in stalls.values() if v == v)
        top = sorted(stalls.items(), key=lambda x: -x[1])[:7]
        if tot:
            out.append("| stall samples (top) | " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top) + " |")
        out.append("")
    return "\n".join(out)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("kind", choices=["launches", "full"])
    p.add_argument("path")
    p.add_argument("--last", type=int, default=0, help="only the last K launches (one step)")
    p.add_argument("--bytes", action="append", default=[], help="kernel-substring=algorithmic GB")
    a = p.parse_args()
    if a.kind == "launches":
        algo = {k: float(v) for k, v in (s.split("=") for s in a.bytes)}
        print(launches(a.path, a.last, algo))
    else:
        print(full(a.path))


if __name__ == "__main__":
    sys.exit(main())
