"""GPU parity of the FP32 solver (pm_*_f32; the paper's FP32 experiments,
PAPER.md:243-274) against the CPU oracle.

The oracle solves the same FP32 inputs (promoted exactly to FP64) in FP64 --
Thomas, pinned to LAPACK dgtsv in test_oracle.py -- so the comparison
measures the FP32 solver's own rounding.  Bars (FP32, unit roundoff
6e-8, diagonally dominant synthetic systems with margin >= 1):
  max relative error ||x - x_ref||_inf / ||x_ref||_inf <= 1e-5
  relative residual ||A x - d||_2 / ||d||_2 (FP64 on the FP32 inputs) <= 1e-5
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

REL_TOL32 = 1e-5
RES_TOL32 = 1e-5


def _f32_system(n, seed):
    return [v.astype(np.float32) for v in oracle.generate(n, seed)]


def _check32(x32, a32, b32, c32, d32):
    a, b, c, d = (np.ascontiguousarray(v, np.float64) for v in (a32, b32, c32, d32))
    a = a.copy()
    c = c.copy()
    a[0] = 0.0
    c[-1] = 0.0
    xref = oracle.thomas(a, b, c, d)
    x = np.ascontiguousarray(x32, np.float64)
    err = oracle.rel_err(x, xref)
    res = oracle.residual(a, b, c, d, x)
    assert err <= REL_TOL32, f"rel err {err:.3e}"
    assert res <= RES_TOL32, f"residual {res:.3e}"
    return err, res


@pytest.mark.parametrize("n", [1, 5, 1000, 12345])
def test_f32_generator_is_rounded_f64(solver, n):
    import torch

    a, b, c, d = solver.generate_device(n, 7, dtype=torch.float32)
    ref = _f32_system(n, 7)
    for t, r in zip((a, b, c, d), ref):
        got = t.cpu().numpy()
        if t is a:
            got, r = got[1:], r[1:]
        if t is c:
            got, r = got[:-1], r[:-1]
        assert np.array_equal(got, r)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 9, 10, 11, 319, 320, 321, 322, 323, 324, 1279, 1281, 4097,
                               100_003, 1_000_000, 3_333_333])
def test_f32_device_solve_m10(solver, n):
    import torch

    a, b, c, d = _f32_system(n, 3)
    t = [torch.from_numpy(v).cuda() for v in (a, b, c, d)]
    x = solver.solve_device(*t, m=10)
    solver.check()
    assert x.dtype == torch.float32
    _check32(x.cpu().numpy(), a, b, c, d)


@pytest.mark.parametrize("m", [2, 3, 4, 7, 8, 16, 17, 33, 64])
@pytest.mark.parametrize("n", [7, 54_321, 400_001])
def test_f32_m_sweep(solver, m, n):
    import torch

    a, b, c, d = _f32_system(n, m)
    t = [torch.from_numpy(v).cuda() for v in (a, b, c, d)]
    x = solver.solve_device(*t, m=m)
    solver.check()
    _check32(x.cpu().numpy(), a, b, c, d)


def test_f32_full_size_n8e7(solver):
    import torch

    n = 80_000_000
    a, b, c, d = solver.generate_device(n, 42, dtype=torch.float32)
    x = solver.solve_device(a, b, c, d, m=10)
    solver.check()
    xh = x.cpu().numpy()
    ah, bh, ch, dh = (t.cpu().numpy() for t in (a, b, c, d))
    del a, b, c, d, x
    torch.cuda.empty_cache()
    _check32(xh, ah, bh, ch, dh)


@pytest.mark.parametrize("ns", [0, 1, 4, 32])
@pytest.mark.parametrize("n", [1000, 2_500_001])
def test_f32_host_streams(solver, ns, n):
    from paper_2501_05938_b200 import pinned_empty

    a, b, c, d = _f32_system(n, 11)
    host = [pinned_empty(n, np.float32) for _ in range(5)]
    for h, v in zip(host, (a, b, c, d)):
        h[:] = v
    x = solver.solve_host(*host[:4], m=10, num_streams=ns, out=host[4])
    assert x.dtype == np.float32
    _check32(x, a, b, c, d)


@pytest.mark.parametrize("nps,batch,m", [(1000, 16, 10), (100_000, 8, 10), (257, 33, 8)])
def test_f32_batch(solver, nps, batch, m):
    import torch

    rng = np.random.default_rng(nps)
    systems = [_f32_system(nps, int(s)) for s in rng.integers(0, 2**31, batch)]
    cat = [np.concatenate([s[k] for s in systems]) for k in range(4)]
    t = [torch.from_numpy(v).cuda() for v in cat]
    x = solver.solve_batch_device(*t, n_per_system=nps, m=m).cpu().numpy()
    solver.check()
    for k, s in enumerate(systems):
        _check32(x[k * nps:(k + 1) * nps], *s)


@pytest.mark.parametrize("fused", [1, 2])
@pytest.mark.parametrize("world", [2, 3])
def test_f32_dist_virtual_ranks(solver, world, fused):
    """fused = 2: the ranks' upper levels in two launches where they apply
    (PM_OPT_UPPER_FUSED; FP32 level 0 uses pair tiles of 64 m rows)."""
    import torch

    from paper_2501_05938_b200 import PartitionSolver
    from paper_2501_05938_b200.dist import split_rows
    from paper_2501_05938_b200.solver import PM_OPT_UPPER_FUSED

    n, m = 1_000_003 if fused == 1 else 2_600_007, 10
    handles = [solver] + [PartitionSolver(0) for _ in range(world - 1)]
    for h in handles:
        h.set_option(PM_OPT_UPPER_FUSED, fused)
    a, b, c, d = _f32_system(n, 5)
    rows = split_rows(n, world, m)
    offs = np.concatenate([[0], np.cumsum(rows)])
    loc = [[torch.from_numpy(v[offs[r]:offs[r + 1]].copy()).cuda() for v in (a, b, c, d)]
           for r in range(world)]
    iface_all = torch.zeros(8 * world, dtype=torch.float32, device="cuda")
    for r in range(world):
        handles[r].dist_reduce(*loc[r], m=m, rank=r, world=world, iface=iface_all[8 * r:8 * r + 8])
    xs = []
    for r in range(world):
        x = torch.empty(rows[r], dtype=torch.float32, device="cuda")
        handles[r].dist_solve(*loc[r], x, m=m, rank=r, world=world, iface_all=iface_all)
        xs.append(x)
    for h in handles:
        h.check()
    solver.set_option(PM_OPT_UPPER_FUSED, 1)
    for h in handles[1:]:
        h.close()
    _check32(torch.cat(xs).cpu().numpy(), a, b, c, d)


def test_f32_zero_pivot(solver):
    import torch

    from paper_2501_05938_b200 import errors

    a, b, c, d = _f32_system(10_000, 1)
    a[55] = b[55] = c[55] = 0.0
    t = [torch.from_numpy(v).cuda() for v in (a, b, c, d)]
    solver.solve_device(*t, m=10)
    with pytest.raises(errors.ComputationError):
        solver.check()


def test_f32_dtype_mismatch_rejected(solver):
    import torch

    from paper_2501_05938_b200 import errors

    a, b, c, d = _f32_system(100, 1)
    t = [torch.from_numpy(v).cuda() for v in (a, b, c, d)]
    t[0] = t[0].double()
    with pytest.raises(errors.ValidationError):
        solver.solve_device(*t, m=10)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_f32_p2p_mixed_precision_session(solver, world):
    """P2P exchange in a session that mixes precisions: an FP64
    solve (the DistributedSolver self-test runs one), then FP32 solves on both
    buffer parities, then FP64 again.  The epoch flags live at a fixed byte
    offset, so FP64 slot data is never read as an FP32 session's flags."""
    import torch

    from paper_2501_05938_b200 import PartitionSolver
    from paper_2501_05938_b200.dist import split_rows

    handles = [solver] + [PartitionSolver(0) for _ in range(world - 1)]
    bufs = [h.dist_exchange_alloc(world) for h in handles]
    for r, h in enumerate(handles):
        h.dist_set_peers(bufs, r)
    n, m = 200_003, 10
    rows = split_rows(n, world, m)
    offs = np.concatenate([[0], np.cumsum(rows)])
    sys64 = oracle.generate(n, 31)
    sys32 = _f32_system(n, 31)

    def run(system, dt):
        loc = [[torch.from_numpy(np.ascontiguousarray(v[offs[r]:offs[r + 1]])).cuda() for v in system]
               for r in range(world)]
        for r in range(world):
            handles[r].dist_reduce_p2p(*loc[r], m=m)
        xs = []
        for r in range(world):
            x = torch.empty(rows[r], dtype=dt, device="cuda")
            handles[r].dist_solve_p2p(*loc[r], x, m=m)
            xs.append(x)
        for h in handles:
            h.check()
        return torch.cat(xs).cpu().numpy()

    for dt in (torch.float64, torch.float32, torch.float32, torch.float32, torch.float64):
        if dt == torch.float64:
            a, b, c, d = sys64
            x = run(sys64, dt)
            xref = oracle.thomas(a, b, c, d)
            assert oracle.rel_err(x, xref) <= 1e-10 and oracle.residual(a, b, c, d, x) <= 1e-12
        else:
            _check32(run(sys32, dt), *sys32)
    for h in handles[1:]:
        h.close()
