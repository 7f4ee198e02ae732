"""CPU tests: the oracle is pinned before anything is checked against it.

Pins: LAPACK dgtsv (third-party, scipy) and the committed
fixtures in tests/golden/ (tests/golden/make_golden.py).  The reference has
no solver golden vectors, so solver parity is "unpinned" by the reference
itself; see DESIGN.md "Oracle".
"""
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("n,seed", [(1, 42), (2, 42), (3, 1), (17, 7), (1000, 42), (100_003, 1_234_567)])
def test_generator_c_matches_numpy(n, seed):
    for x, y in zip(oracle.generate(n, seed), oracle.generate_np(n, seed)):
        assert np.array_equal(x, y)


def test_generator_golden():
    g = np.load(GOLD / "generator.npz")
    for n, seed in [(1, 42), (2, 42), (17, 7), (1000, 42), (100003, 1234567)]:
        arrs = oracle.generate(n, seed)
        for name, v in zip("abcd", arrs):
            assert np.array_equal(v[:8], g[f"n{n}_s{seed}_{name}_head"])
            assert np.array_equal(v[-8:], g[f"n{n}_s{seed}_{name}_tail"])


def test_generator_properties():
    a, b, c, d = oracle.generate(50_000, 3)
    assert a[0] == 0.0 and c[-1] == 0.0
    assert np.all(np.abs(b) >= np.abs(a) + np.abs(c) + 1.0)  # strict dominance, margin >= 1
    assert np.all(np.abs(a) < 1) and np.all(np.abs(c) < 1) and np.all(np.abs(d) < 1)
    assert 0.45 < np.mean(b > 0) < 0.55


def test_solvers_against_golden_dgtsv():
    s = np.load(GOLD / "systems.npz")
    for key in s.files:
        a, b, c, d, xg = (np.ascontiguousarray(v) for v in s[key])
        xt = oracle.thomas(a, b, c, d)
        assert oracle.rel_err(xt, xg) < 1e-13, key
        for m in (2, 3, 10, 64):
            xp = oracle.partition_solve(a, b, c, d, m)
            assert oracle.rel_err(xp, xg) < 1e-12, (key, m)
            assert oracle.residual(a, b, c, d, xp) < 1e-12, (key, m)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 10, 11, 19, 20, 21, 999, 10_001])
@pytest.mark.parametrize("m", [2, 3, 4, 7, 10, 16, 128])
def test_partition_matches_dgtsv_live(n, m):
    a, b, c, d = oracle.generate(n, n * 31 + m)
    xr = oracle.dgtsv(a, b, c, d)
    x = oracle.partition_solve(a, b, c, d, m)
    assert oracle.rel_err(x, xr) < 1e-13
    assert oracle.residual(a, b, c, d, x) < 1e-14


def test_thomas_python_mirror():
    a, b, c, d = oracle.generate(257, 9)
    assert oracle.rel_err(oracle.thomas_np(a, b, c, d), oracle.thomas(a, b, c, d)) < 1e-15


def test_ignored_corners():
    a, b, c, d = oracle.generate(100, 5)
    x = oracle.thomas(a, b, c, d)
    a2, c2 = a.copy(), c.copy()
    a2[0], c2[-1] = 1e3, -1e3
    assert np.array_equal(oracle.partition_solve(a2, b, c2, d, 10), oracle.partition_solve(a, b, c, d, 10))
    assert oracle.rel_err(oracle.partition_solve(a2, b, c2, d, 10), x) < 1e-14


def test_zero_pivot_detected():
    a, b, c, d = oracle.generate(30, 1)
    b = b.copy()
    b[0] = 0.0
    with pytest.raises(ArithmeticError):
        oracle.thomas(a, b, c, d)


def test_checkers():
    x = np.array([1.0, -2.0, 4.0])
    assert oracle.rel_err(x, x) == 0.0
    assert abs(oracle.rel_err(x + np.array([0.0, 0.0, 0.4]), x) - 0.1) < 1e-15
    a, b, c, d = oracle.generate(1000, 2)
    xr = oracle.dgtsv(a, b, c, d)
    assert oracle.residual(a, b, c, d, xr) < 1e-15
    assert oracle.residual(a, b, c, d, np.zeros(1000)) == pytest.approx(1.0)


@pytest.mark.parametrize("n,row0,count", [(1000, 0, 1000), (1000, 999, 1), (123_457, 40_000, 50_001)])
def test_generate_range_is_a_slice(n, row0, count):
    full = oracle.generate(n, 9)
    for x, y in zip(oracle.generate_range(n, row0, count, 9), full):
        assert np.array_equal(x, y[row0:row0 + count])


@pytest.mark.parametrize("n,chunk", [(1, 1 << 18), (5, 2), (2_000_003, 100_000), (300_000, 4096)])
def test_windowed_check_equals_whole_system_thomas(n, chunk):
    """orc_check_generated (windowed Thomas, pad 1024) reproduces the
    whole-system Thomas solution bit for bit on the generated systems, so a
    solution checked by windows is checked against Thomas itself."""
    a, b, c, d = oracle.generate(n, 11)
    x = oracle.thomas(a, b, c, d)
    r = oracle.check_generated(x, n, 0, 11, chunk=chunk)
    assert r["max_err"] == 0.0
    assert abs(r["residual"] - oracle.residual(a, b, c, d, x)) <= 1e-3 * r["residual"] + 1e-30
    # a slice with its halo values, and a perturbation is seen by both bars
    lo, hi = n // 3, max(n // 3 + 1, 2 * n // 3)
    xl = x[lo - 1] if lo > 0 else 0.0
    xr = x[hi] if hi < n else 0.0
    assert oracle.check_generated(x[lo:hi], n, lo, 11, xl, xr, chunk=chunk)["max_err"] == 0.0
    xp = x.copy()
    xp[n // 2] += 1e-7
    rp = oracle.check_generated(xp, n, 0, 11, chunk=chunk)
    assert rp["rel_err"] > 1e-8 and rp["residual"] > 1e-13


def test_windowed_check_combines_over_ranks():
    n = 1_000_000
    a, b, c, d = oracle.generate(n, 12)
    x = oracle.thomas(a, b, c, d)
    cuts = [0, 250_000, 600_010, n]
    parts = [oracle.check_generated(x[lo:hi], n, lo, 12, x[lo - 1] if lo else 0.0, x[hi] if hi < n else 0.0)
             for lo, hi in zip(cuts[:-1], cuts[1:])]
    r = oracle.finish_check(parts)
    assert r["rel_err"] == 0.0
    assert abs(r["residual"] - oracle.residual(a, b, c, d, x)) <= 1e-3 * r["residual"]
