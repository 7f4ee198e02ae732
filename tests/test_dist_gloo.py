"""World-size-2 gloo test of the row-sharded solve's host protocol (CPU).

The device kernels cannot run here, so each rank uses a numpy stand-in for
pm_dist_reduce_f64 / pm_dist_solve_f64 (test infrastructure: the same
segment algebra and chain solve, dense for small sizes); what is under test is
the product's host logic -- split_rows, DistributedSolver's reduce ->
all_gather -> solve ordering and the 8-double interface layout
[Fa, La, Fb, Lb, Fc, Lc, Fd, Ld] -- over a real torch.distributed group.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class NumpyDistBackend:
    """Stand-in for the CUDA solver's dist_reduce / dist_solve."""

    device = "cpu"

    @staticmethod
    def _interior(a, b, c, d, xs, xe):
        n = len(b)
        if n <= 2:
            return np.array([xs, xe][:n])
        A = np.diag(b[1:-1]) + np.diag(a[2:-1], -1) + np.diag(c[1:-2], 1)
        r = d[1:-1].copy()
        r[0] -= a[1] * xs
        r[-1] -= c[-2] * xe
        return np.concatenate([[xs], np.linalg.solve(A, r), [xe]])

    def dist_reduce(self, a, b, c, d, m, rank, world, iface, stream=None):
        a, b, c, d = (t.numpy().copy() for t in (a, b, c, d))
        if rank == 0:
            a[0] = 0.0
        if rank == world - 1:
            c[-1] = 0.0
        n = len(b)
        # x_interior = y - g*x0 - h*x_{n-1}
        y = self._interior(a, b, c, d, 0.0, 0.0)
        g = self._interior(a, b, c, np.zeros(n), 1.0, 0.0)
        h = self._interior(a, b, c, np.zeros(n), 0.0, 1.0)
        # row 0: a0 x_{-1} + b0 x0 + c0 x1 ; x1 = y1 + g1 x0 + h1 x_{n-1}  (signs folded into g/h)
        F = [a[0], b[0] + c[0] * g[1], c[0] * h[1], d[0] - c[0] * y[1]]
        L = [a[-1] * g[-2], b[-1] + a[-1] * h[-2], c[-1], d[-1] - a[-1] * y[-2]]
        iface[:] = torch.tensor([F[0], L[0], F[1], L[1], F[2], L[2], F[3], L[3]], dtype=torch.float64)

    def dist_solve(self, a, b, c, d, x, m, rank, world, iface_all, stream=None):
        f = iface_all.numpy().reshape(world, 8)
        # 2*world-row interface system in unknowns (x_first_r, x_last_r)
        nr = 2 * world
        A = np.zeros((nr, nr))
        r = np.zeros(nr)
        for k in range(world):
            Fa, La, Fb, Lb, Fc, Lc, Fd, Ld = f[k]
            i = 2 * k
            if k > 0:
                A[i, i - 1] = Fa
            A[i, i], A[i, i + 1], r[i] = Fb, Fc, Fd
            A[i + 1, i], A[i + 1, i + 1], r[i + 1] = La, Lb, Ld
            if k < world - 1:
                A[i + 1, i + 2] = Lc
        xi = np.linalg.solve(A, r)
        aa, bb, cc, dd = (t.numpy().copy() for t in (a, b, c, d))
        x[:] = torch.from_numpy(self._interior(aa, bb, cc, dd, xi[2 * rank], xi[2 * rank + 1]))


def _worker(rank, world, port, n, m, q, exchange="collective"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2501_05938_b200.dist import DistributedSolver, row_offset, split_rows

        rows = split_rows(n, world, m)
        off = row_offset(n, world, m, rank)
        a, b, c, d = (torch.from_numpy(v[off:off + rows[rank]].copy()) for v in oracle.generate(n, 5))
        ds = DistributedSolver(NumpyDistBackend(), device=torch.device("cpu"), exchange=exchange)
        # "auto": the peer-memory setup cannot succeed without CUDA; every rank
        # still joins the same collectives and all agree on the all-gather
        assert ds.exchange == "collective"
        x = torch.empty(rows[rank], dtype=torch.float64)
        ds.solve(a, b, c, d, x, m=m)
        mx = max(rows)
        padded = torch.zeros(mx, dtype=torch.float64)
        padded[:rows[rank]] = x
        parts = [torch.empty(mx, dtype=torch.float64) for _ in rows]
        dist.all_gather(parts, padded)
        if rank == 0:
            xs = torch.cat([p[:k] for p, k in zip(parts, rows)]).numpy()
            ah, bh, ch, dh = oracle.generate(n, 5)
            q.put(float(oracle.rel_err(xs, oracle.thomas(ah, bh, ch, dh))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["collective", "auto"])
@pytest.mark.parametrize("n,m,world", [(200, 10, 2), (157, 7, 2), (64, 4, 3)])
def test_row_sharded_protocol_gloo(n, m, world, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) < 1e-12


def test_split_rows():
    from paper_2501_05938_b200.dist import split_rows

    assert split_rows(100, 1, 10) == [100]
    r = split_rows(8 * 10**7 * 8, 8, 10)
    assert sum(r) == 8 * 10**7 * 8 and all(k % 10 == 0 for k in r[:-1])
    r = split_rows(1001, 3, 10)
    assert r[:2] == [330, 330] and r[2] == 341
    from paper_2501_05938_b200 import ValidationError

    with pytest.raises(ValidationError):
        split_rows(15, 3, 10)
