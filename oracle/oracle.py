"""ctypes wrappers of the oracle C library plus numpy restatements.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Parity status: the reference ships no solver,
hence no solver golden vectors -- "parity unpinned" by the reference itself.
The restatement is pinned to LAPACK ``dgtsv`` (scipy 1.18.1, a third-party
solver, not a reference dependency) and to committed fixtures under
``tests/golden/``.  The stream-count side is pinned to the reference's own
header through ``oracle/_ref/libstreamtune_ref.so``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle_tridiag.so"
REF_PATH = HERE / "_ref" / "libstreamtune_ref.so"

__all__ = [
    "build_oracle", "lib", "ref_lib", "generate", "generate_np", "thomas", "partition_solve",
    "residual", "rel_err", "dgtsv", "thomas_np", "max_threads", "generate_range", "check_generated",
    "finish_check",
]

_lib = None
_ref = None
_D = C.POINTER(C.c_double)


def build_oracle() -> None:
    """Builds liboracle_tridiag.so and, when /root/reference exists, _ref/."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build_oracle()
        L = C.CDLL(str(LIB_PATH))
        L.orc_generate.argtypes = [_D, _D, _D, _D, C.c_int64, C.c_uint64]
        L.orc_generate.restype = None
        L.orc_generate_range.argtypes = [_D, _D, _D, _D, C.c_int64, C.c_int64, C.c_int64, C.c_uint64]
        L.orc_generate_range.restype = None
        L.orc_check_generated.argtypes = [_D, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_double,
                                          C.c_double, C.c_int64, C.c_int64, _D]
        L.orc_check_generated.restype = C.c_int
        L.orc_thomas.argtypes = [_D, _D, _D, _D, _D, _D, C.c_int64]
        L.orc_thomas.restype = C.c_int
        L.orc_partition_workspace.argtypes = [C.c_int64, C.c_int32]
        L.orc_partition_workspace.restype = C.c_int64
        L.orc_partition_solve.argtypes = [_D, _D, _D, _D, _D, C.c_int64, C.c_int32, _D, C.c_int]
        L.orc_partition_solve.restype = C.c_int
        L.orc_residual.argtypes = [_D, _D, _D, _D, _D, C.c_int64]
        L.orc_residual.restype = C.c_double
        L.orc_rel_err.argtypes = [_D, _D, C.c_int64]
        L.orc_rel_err.restype = C.c_double
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def ref_lib():
    """The reference's timing_model.hpp compiled in place (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            build_oracle()
        if not REF_PATH.exists():
            raise FileNotFoundError(f"{REF_PATH} missing (reference tree absent when built)")
        R = C.CDLL(str(REF_PATH))
        R.ref_stream_count_is_valid.argtypes = [C.c_int]
        R.ref_stream_count_is_valid.restype = C.c_int
        R.ref_total_unstreamed.argtypes = [_D]
        R.ref_total_unstreamed.restype = C.c_double
        R.ref_overlap_sum.argtypes = [_D]
        R.ref_overlap_sum.restype = C.c_double
        R.ref_streamed_lower_bound.argtypes = [_D, C.c_int, C.c_double, _D]
        R.ref_streamed_lower_bound.restype = C.c_int
        R.ref_overhead_from_measurement.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, _D]
        R.ref_overhead_from_measurement.restype = C.c_int
        R.ref_overlap_benefit.argtypes = [C.c_int, C.c_double, C.c_double, _D]
        R.ref_overlap_benefit.restype = C.c_int
        R.ref_validate_stage_timings.argtypes = [_D, C.c_ulonglong, C.c_char_p, C.c_int]
        R.ref_validate_stage_timings.restype = C.c_int
        R.ref_streamed_run_validate.argtypes = [C.c_ulonglong, C.c_int, C.c_double, C.c_char_p, C.c_int]
        R.ref_streamed_run_validate.restype = C.c_int
        _ref = R
    return _ref


def _p(x: np.ndarray):
    assert x.dtype == np.float64 and x.flags.c_contiguous
    return x.ctypes.data_as(_D)


def max_threads() -> int:
    return int(lib().orc_max_threads())


def generate(n: int, seed: int = 42):
    """Counter-based synthetic system (identical bits to pm_generate_f64)."""
    a, b, c, d = (np.empty(n, np.float64) for _ in range(4))
    lib().orc_generate(_p(a), _p(b), _p(c), _p(d), n, seed)
    return a, b, c, d


def generate_range(n_total: int, row0: int, count: int, seed: int = 42):
    """Rows [row0, row0 + count) of the n_total-row generated system."""
    a, b, c, d = (np.empty(count, np.float64) for _ in range(4))
    lib().orc_generate_range(_p(a), _p(b), _p(c), _p(d), n_total, row0, count, seed)
    return a, b, c, d


def check_generated(x, n_total: int, row0: int = 0, seed: int = 42, xl: float = 0.0, xr: float = 0.0,
                    chunk: int = 1 << 18, pad: int = 1024) -> dict:
    """Windowed Thomas check of x = rows [row0, row0+len(x)) of the generated
    system (orc_check_generated): no copy of the system is held.  Returns the
    parts of the two bars so ranks can combine them:
    rel_err = max_err / max_ref (max over ranks), residual =
    sqrt(sum rsq / sum dsq) (sums over ranks)."""
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(4, np.float64)
    st = lib().orc_check_generated(_p(x), n_total, row0, len(x), seed, float(xl), float(xr), chunk, pad,
                                   _p(out))
    if st != 0:
        raise ArithmeticError(f"oracle windowed check failed with status {st}")
    r = {"max_err": float(out[0]), "max_ref": float(out[1]), "rsq": float(out[2]), "dsq": float(out[3])}
    return finish_check([r])


def finish_check(parts) -> dict:
    """Combine per-rank check_generated parts into the two bars."""
    me = max(p["max_err"] for p in parts)
    mr = max(p["max_ref"] for p in parts)
    rs = sum(p["rsq"] for p in parts)
    ds = sum(p["dsq"] for p in parts)
    return {"max_err": me, "max_ref": mr, "rsq": rs, "dsq": ds,
            "rel_err": me / mr if mr > 0 else me, "residual": float(np.sqrt(rs / ds)) if ds > 0 else float(np.sqrt(rs))}


# ---- numpy restatement of the generator (cross-checks the C one) -------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _key(seed: int, arr: int) -> np.uint64:
    with np.errstate(over="ignore"):
        v = np.uint64(seed) ^ (np.uint64(0x632BE59BD9B4E019) * np.uint64(arr + 1))
    return _splitmix64(np.array([v], dtype=np.uint64))[0]


def generate_np(n: int, seed: int = 42):
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = [(_splitmix64(_key(seed, k) + i) >> np.uint64(11)).astype(np.float64) * 2.0**-53
             for k in range(4)]
        sgn = _splitmix64(_key(seed, 4) + i) >> np.uint64(63)
    a = 2.0 * u[0] - 1.0
    c = 2.0 * u[1] - 1.0
    if n:
        a[0] = 0.0
        c[n - 1] = 0.0
    mag = ((np.abs(a) + np.abs(c)) + 1.0) + u[2]
    b = np.where(sgn == 1, -mag, mag)
    d = 2.0 * u[3] - 1.0
    return a, b, c, d


# ---- solvers -------------------------------------------------------------------
def thomas(a, b, c, d):
    n = len(b)
    x = np.empty(n, np.float64)
    w = np.empty(n, np.float64)
    st = lib().orc_thomas(_p(a), _p(b), _p(c), _p(d), _p(x), _p(w), n)
    if st != 0:
        raise ArithmeticError(f"oracle Thomas failed with status {st}")
    return x


def partition_solve(a, b, c, d, m: int = 10, threads: int = 0):
    """The paper's partition method (Stage 1 / serial Stage 2 / Stage 3)."""
    n = len(b)
    ws = np.empty(max(1, lib().orc_partition_workspace(n, m)), np.float64)
    x = np.empty(n, np.float64)
    st = lib().orc_partition_solve(_p(a), _p(b), _p(c), _p(d), _p(x), n, m, _p(ws), threads)
    if st != 0:
        raise ArithmeticError(f"oracle partition solve failed with status {st}")
    return x


def thomas_np(a, b, c, d):
    """Pure-Python Thomas (small cases only)."""
    n = len(b)
    cp = np.zeros(n)
    x = np.zeros(n)
    cp[0] = (c[0] if n > 1 else 0.0) / b[0]
    x[0] = d[0] / b[0]
    for i in range(1, n):
        den = b[i] - a[i] * cp[i - 1]
        cp[i] = (c[i] if i < n - 1 else 0.0) / den
        x[i] = (d[i] - a[i] * x[i - 1]) / den
    for i in range(n - 2, -1, -1):
        x[i] -= cp[i] * x[i + 1]
    return x


def dgtsv(a, b, c, d):
    """LAPACK dgtsv (scipy / OpenBLAS): the third-party pin of the oracle."""
    from scipy.linalg import lapack

    n = len(b)
    if n == 1:
        return np.array([d[0] / b[0]])
    _, _, _, x, info = lapack.dgtsv(a[1:].copy(), b.copy(), c[:-1].copy(), d.copy())
    if info != 0:
        raise ArithmeticError(f"dgtsv info={info}")
    return x


def residual(a, b, c, d, x) -> float:
    return float(lib().orc_residual(_p(a), _p(b), _p(c), _p(d), _p(x), len(b)))


def rel_err(x, xref) -> float:
    return float(lib().orc_rel_err(_p(x), _p(xref), len(x)))
