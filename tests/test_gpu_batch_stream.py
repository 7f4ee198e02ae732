"""GPU parity of the batch tile-stream kernel (csrc/pm_batch_stream.cu,
PM_OPT_BATCH_CLUSTER = 2) against the CPU oracle.

Same bars as test_gpu_parity.py (BASELINE.json north_star): max relative
error <= 1e-10 against the oracle's Thomas solve of each system, relative
residual <= 1e-12.  Small grids (PM_OPT_MAX_CTAS, PM_OPT_BATCH_WARPS) put
many rounds on every warp, so the lag / ring / per-system flag machinery is
exercised at test sizes; ragged last tiles, one-tile systems, every compiled
m, back-to-back launches (flags and counters must return to zero), x = d
aliasing and the zero-pivot error path are covered.
"""
import numpy as np
import pytest

import oracle
from test_gpu_parity import _batch_systems, _check

pytestmark = pytest.mark.gpu


def _opts(solver, **kw):
    from paper_2501_05938_b200 import solver as S

    names = {"kernel": S.PM_OPT_BATCH_CLUSTER, "ctas": S.PM_OPT_MAX_CTAS, "warps": S.PM_OPT_BATCH_WARPS,
             "stages": S.PM_OPT_BATCH_STAGES, "lag": S.PM_OPT_BATCH_LAG, "discard": S.PM_OPT_BATCH_DISCARD}
    for k, v in kw.items():
        solver.set_option(names[k], v)


def _reset(solver):
    _opts(solver, kernel=0, ctas=0, warps=0, stages=0, lag=0, discard=15)


def _solve(solver, cat, nps, m, out=None, **kw):
    import torch

    t = [torch.from_numpy(v).cuda() for v in cat]
    _opts(solver, kernel=2, **kw)
    try:
        x = solver.solve_batch_device(*t, n_per_system=nps, m=m, out=t[3] if out == "d" else None)
        solver.check()
        plan = solver.last_batch_plan()
    finally:
        _reset(solver)
    return x.cpu().numpy(), plan


@pytest.mark.parametrize("nps,batch,m", [
    (100_000, 12, 10), (640, 40, 10), (642, 37, 10), (20_002, 13, 10), (99_998, 5, 8), (4_096, 31, 2),
    (65_536, 6, 16), (320, 50, 10), (2, 300, 2), (16, 64, 8), (1_000_000, 2, 10), (5_000, 9, 10)])
@pytest.mark.parametrize("ctas,warps,lag", [(1, 2, 3), (3, 4, 5), (7, 8, 0)])
def test_stream_kernel_parity(solver, nps, batch, m, ctas, warps, lag):
    systems, cat = _batch_systems(nps, batch, nps * 13 + batch + ctas)
    x, plan = _solve(solver, cat, nps, m, ctas=ctas, warps=warps, lag=lag)
    tps = -(-nps // (32 * m))
    nw = ctas * warps
    lag_min = max(lag or 4, -(-(tps - 1) // nw) + 1)  # the lag covers a system's rounds
    if plan["kernel"] == "stream":
        sp = plan["stream"]
        assert sp["tps"] == tps and sp["ctas"] == ctas and sp["lag"] >= sp["stages"] + 1
        assert sp["lag"] >= lag_min
    else:  # lag > 64 rounds, fewer rounds per warp than the lag, or the system's
        # segments do not fit shared memory beside the stages: level kernels
        assert lag_min > 64 or batch * tps // nw < lag_min or tps * 64 > 64 * 1024, plan
    for k, s in enumerate(systems):
        _check(x[k * nps:(k + 1) * nps], *s)


@pytest.mark.parametrize("stages", [1, 2])
@pytest.mark.parametrize("discard", list(range(16)))
def test_stream_kernel_stages_discard(solver, stages, discard):
    """Option bits: 1 discard consumed node lines, 2 L2 hints, 4 early issue
    (one stage per warp), 8 out-of-order publication by the control warp."""
    nps, batch, m = 12_000, 40, 10
    systems, cat = _batch_systems(nps, batch, 5 + stages)
    x, plan = _solve(solver, cat, nps, m, ctas=5, warps=6, stages=stages, discard=discard)
    assert plan["kernel"] == "stream" and plan["stream"]["stages"] == stages, plan
    for k, s in enumerate(systems):
        _check(x[k * nps:(k + 1) * nps], *s)


def _counters(solver, n):
    import ctypes as C

    from paper_2501_05938_b200 import _lib

    buf = (C.c_uint32 * n)()
    assert _lib.load().pm_batch_stream_counters(solver._h, buf, n) == 0
    return np.array(buf[:])


def test_stream_kernel_back_to_back(solver):
    """Launches in a row on one handle with different data, batch sizes and
    plans: the per-system flags and counters must be back at zero after every
    launch (a layout change once let ring data land on them)."""
    import torch

    cases = [(3_200, 64, 10), (20_002, 13, 10), (4_096, 31, 2), (3_200, 64, 10), (640, 90, 10),
             (20_002, 13, 10), (4_096, 31, 2)]
    outs = []
    _opts(solver, kernel=2, ctas=4, warps=4, lag=3)
    try:
        for rep, (nps, batch, m) in enumerate(cases):
            systems, cat = _batch_systems(nps, batch, 100 + rep)
            t = [torch.from_numpy(v).cuda() for v in cat]
            x = solver.solve_batch_device(*t, n_per_system=nps, m=m)
            solver.check()
            assert solver.last_batch_plan()["kernel"] == "stream"
            assert not _counters(solver, 3 * 32 * batch).any()
            outs.append((systems, x, nps))
    finally:
        _reset(solver)
    for systems, x, nps in outs:
        xh = x.cpu().numpy()
        for k, s in enumerate(systems):
            _check(xh[k * nps:(k + 1) * nps], *s)


def test_stream_kernel_aliasing_and_zero_pivot(solver):
    from paper_2501_05938_b200 import errors

    nps, batch = 20_000, 16
    systems, cat = _batch_systems(nps, batch, 11)
    x, plan = _solve(solver, cat, nps, 10, out="d", ctas=4, warps=4)
    assert plan["kernel"] == "stream"
    for k, s in enumerate(systems):
        _check(x[k * nps:(k + 1) * nps], *s)
    cat[1][3 * nps + 5] = 0.0  # b = 0 inside a block interior of system 3
    cat[0][3 * nps + 5] = 0.0
    cat[2][3 * nps + 5] = 0.0
    with pytest.raises(errors.ComputationError):
        _solve(solver, cat, nps, 10, ctas=4, warps=4)


def test_stream_kernel_row_scaled(solver):
    """Rows scaled over many orders of magnitude: the fast continuant pivots
    may leave the FP range; the retry with classic sweeps must then solve it."""
    nps, batch = 6_400, 20
    systems, cat = _batch_systems(nps, batch, 23)
    rng = np.random.default_rng(1)
    scale = 10.0 ** rng.uniform(-60, 60, nps * batch)
    cat = [v * scale for v in cat]
    systems = [tuple(v[k * nps:(k + 1) * nps].copy() for v in cat) for k in range(batch)]
    for s in systems:
        s[0][0] = 0.0
        s[2][-1] = 0.0
    x, _ = _solve(solver, cat, nps, 10, ctas=3, warps=4)
    for k, s in enumerate(systems):
        _check(x[k * nps:(k + 1) * nps], *s)


def test_batch_config4_stream_kernel(solver):
    """BASELINE config 4 (4096 x 1e5) through the tile-stream kernel on the
    full grid, sampled systems checked against the oracle."""
    import torch
    from paper_2501_05938_b200.solver import PM_OPT_BATCH_CLUSTER

    nps, batch = 100_000, 4096
    a, b, c, d = solver.generate_device(nps * batch, 99)
    solver.set_option(PM_OPT_BATCH_CLUSTER, 2)
    try:
        x = solver.solve_batch_device(a, b, c, d, n_per_system=nps, m=10)
        solver.check()
        plan = solver.last_batch_plan()
    finally:
        solver.set_option(PM_OPT_BATCH_CLUSTER, 0)
    assert plan["kernel"] == "stream" and plan["stream"]["ctas"] == torch.cuda.get_device_properties(0).multi_processor_count
    xh = x.cpu().numpy()
    for k in (0, 1, 999, 2048, 4095):
        sl = slice(k * nps, (k + 1) * nps)
        sa, sb, sc, sd = (t[sl].cpu().numpy().copy() for t in (a, b, c, d))
        sa[0] = 0.0
        sc[-1] = 0.0
        _check(xh[sl], sa, sb, sc, sd)
