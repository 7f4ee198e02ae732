"""Generates tests/golden/*.npz -- committed fixtures pinning the CPU oracle.

The reference ships no solver and no solver vectors, so the
solver fixtures are solved by LAPACK dgtsv (scipy.linalg.lapack, OpenBLAS),
an independent third-party implementation; the generator fixture pins the
counter-based input generator (oracle/tridiag_oracle.c, csrc/pm_kernels.cu).
Run from the repo root:  python tests/golden/make_golden.py
"""
from pathlib import Path
import sys

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    # 1) generator: first/last 8 values of every array for a few (n, seed)
    gen = {}
    for n, seed in [(1, 42), (2, 42), (17, 7), (1000, 42), (100003, 1234567)]:
        a, b, c, d = oracle.generate_np(n, seed)
        for name, v in zip("abcd", (a, b, c, d)):
            gen[f"n{n}_s{seed}_{name}_head"] = v[:8]
            gen[f"n{n}_s{seed}_{name}_tail"] = v[-8:]
    np.savez_compressed(OUT / "generator.npz", **gen)

    # 2) solved systems: generator inputs and adversarial-but-dominant ones
    sols = {}
    rng = np.random.default_rng(20250110)
    cases = [(n, s) for n in (1, 2, 3, 4, 9, 10, 11, 64, 319, 320, 321, 1000, 4097) for s in (42,)]
    for n, seed in cases:
        a, b, c, d = oracle.generate_np(n, seed)
        sols[f"gen_n{n}"] = np.stack([a, b, c, d, oracle.dgtsv(a, b, c, d)])
    for k, n in enumerate((5, 50, 500, 3333)):
        a = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-3, 3, n)
        c = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-3, 3, n)
        a[0] = c[-1] = 0.0
        b = (np.abs(a) + np.abs(c)) * rng.uniform(1.01, 3.0, n) + 1e-3
        b *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
        d = rng.normal(size=n) * 10.0 ** rng.integers(-2, 3, n)
        sols[f"scaled_n{n}"] = np.stack([a, b, c, d, oracle.dgtsv(a, b, c, d)])
    np.savez_compressed(OUT / "systems.npz", **sols)
    print("wrote", OUT / "generator.npz", OUT / "systems.npz")


if __name__ == "__main__":
    main()
