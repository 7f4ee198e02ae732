#!/usr/bin/env python
"""Write profiles/ncu_traffic.json from ncu launch lists of THIS build.

bench.py quotes `roofline.traffic` (dram__bytes_read.sum + dram__bytes_write.sum
per launch of the dominant kernel) only when profiles/ncu_traffic.json carries
the kernel build hash of the sources it is running (bench.kernel_build_hash).
This tool reads the CSV launch lists written by

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
      --clock-control none --csv --log-file L.csv python bench.py ...

(scripts/gpu_final_evidence.sh), takes the LAST launch of each kernel of interest
(the last step: warm caches as in the timed region) and stamps the result
with the build hash.

usage: tools/stamp_traffic.py --single launches_single.csv [--batch launches_batch.csv]
                              [--batch-cluster launches_cluster.csv] [--c5 launches_c5.csv]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def _bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1.0)


def per_launch(path: str) -> list[tuple[str, float]]:
    """[(kernel name, dram read+write bytes)] in launch order."""
    text = Path(path).read_text()
    start = text.find('"ID"')
    if start < 0:
        raise SystemExit(f"{path}: no ncu CSV table")
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per: dict[tuple[str, str], float] = {}
    order: list[tuple[str, str]] = []
    for r in rows:
        if r["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        k = (r["ID"], r["Kernel Name"])
        if k not in per:
            order.append(k)
            per[k] = 0.0
        per[k] += _bytes(r["Metric Value"], r["Metric Unit"])
    return [(k[1], per[k]) for k in order]


def last_of(launches, *needles: str):
    hit = [b for name, b in launches if all(n in name for n in needles)]
    return int(hit[-1]) if hit else None


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--single", required=True, help="launch list of bench.py (config 3)")
    p.add_argument("--batch", help="launch list of bench.py --workload batch (level kernels)")
    p.add_argument("--batch-cluster", help="launch list of the batch cluster kernel")
    p.add_argument("--batch-stream", help="launch list of the batch tile-stream kernel")
    p.add_argument("--f32", help="launch list of bench.py --precision f32 (pair-tile kernels)")
    p.add_argument("--out", default=str(ROOT / "profiles" / "ncu_traffic.json"))
    a = p.parse_args()
    doc = {"build_hash": bench.kernel_build_hash(),
           "source": "tools/stamp_traffic.py from ncu launch lists (last launch of each kernel): "
                     + ", ".join(Path(x).name for x in (a.single, a.batch, a.batch_cluster, a.batch_stream, a.f32) if x)}
    s = per_launch(a.single)
    doc["reduce_level0_bytes_per_launch"] = last_of(s, "warp_tile_kernel<10, 0")
    doc["solve_level0_bytes_per_launch"] = last_of(s, "warp_tile_kernel<10, 1")
    if a.batch:
        b = per_launch(a.batch)
        doc["batch_reduce_level0_bytes_per_launch"] = last_of(b, "warp_tile_kernel<10, 0")
        doc["batch_solve_level0_bytes_per_launch"] = last_of(b, "warp_tile_kernel<10, 1")
    if a.batch_cluster:
        c = per_launch(a.batch_cluster)
        doc["batch_cluster_bytes_per_launch"] = last_of(c, "batch_cluster")
    if a.batch_stream:
        c = per_launch(a.batch_stream)
        doc["batch_stream_bytes_per_launch"] = last_of(c, "batch_stream")
    if a.f32:
        f = per_launch(a.f32)
        doc["reduce_level0_f32_bytes_per_launch"] = last_of(f, "warp_pair_kernel<10, 0")
        doc["solve_level0_f32_bytes_per_launch"] = last_of(f, "warp_pair_kernel<10, 1")
    Path(a.out).write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
