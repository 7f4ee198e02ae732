#!/usr/bin/env python
"""SASS instruction histogram of the built solver library, per kernel.

Runs `cuobjdump -sass` on paper_2501_05938_b200/libpm_tridiag.so and counts,
for every kernel whose name matches --kernel (default: the hot kernels), the
opcodes that prove the hardware paths DESIGN.md claims: UBLKCP (cp.async.bulk
global<->shared), SYNCS (mbarrier), SHFL (warp trees), MUFU.RCP64H (FP64
reciprocal seed), DFMA/DMUL/DADD (FP64 pipe), LDS/STS, LDG/STG, and the
tensor-core / TMEM opcodes (UTCMMA/UTCHMMA/LDTM/STTM) that must be absent from
an FP64 streaming solver.  Output: a Markdown table (stdout or --out).
"""
from __future__ import annotations

import argparse
import re
import subprocess
from collections import Counter, OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OPS = ["UBLKCP", "SYNCS", "SHFL", "MUFU.RCP64H", "DFMA", "DMUL", "DADD", "DSETP", "LDS", "STS",
       "LDG", "STG", "ATOM", "RED", "MEMBAR", "BAR", "UTCMMA", "UTCHMMA", "LDTM", "STTM"]
HOT = r"warp_tile_kernel|warp_pair_kernel|upper_fused_kernel|batch_|tile_kernel"


def histogram(lib: Path, pattern: str):
    out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    kernels: "OrderedDict[str, Counter]" = OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1) if re.search(pattern, _demangle(m.group(1))) else None
            if cur:
                kernels[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(1)
        c = kernels[cur]
        c["_total"] += 1
        for k in OPS:
            if op == k or op.startswith(k + "."):
                c[k] += 1
    return kernels


def _demangle(name: str) -> str:
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip() or name
    except OSError:
        return name


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--lib", default=str(ROOT / "paper_2501_05938_b200" / "libpm_tridiag.so"))
    p.add_argument("--kernel", default=HOT)
    p.add_argument("--out")
    a = p.parse_args()
    ks = histogram(Path(a.lib), a.kernel)
    cols = ["_total"] + OPS
    lines = ["| kernel | " + " | ".join("instr" if c == "_total" else c for c in cols) + " |",
             "|---|" + "---|" * len(cols)]
    for name, c in ks.items():
        short = _demangle(name).replace("(anonymous namespace)::", "").split("(")[0]
        lines.append(f"| `{short}` | " + " | ".join(str(c.get(k, 0)) for k in cols) + " |")
    text = "\n".join(lines) + "\n"
    if a.out:
        Path(a.out).write_text(text)
    print(text)


if __name__ == "__main__":
    main()
