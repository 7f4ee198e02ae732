"""Row-sharded single system over ranks (BASELINE.json config 5).

One process per GPU.  Rank r owns the contiguous rows [off_r, off_r + n_r).
The only cross-GPU step is the all-gather of every rank's two interface
equations (8 doubles = 64 B per rank, NCCL over NVLink):

    pm_dist_reduce_f64   Stage 1 + local upper levels -> iface (8 doubles)
    all_gather(iface)    -> iface_all (8 * world doubles, rank order)
    pm_dist_solve_f64    2*world-row interface system (redundant, one thread)
                         -> local Stage 3 of every level -> x

`split_rows` gives every rank but the last a multiple of m rows (the solver
requires it there: a non-last rank's final m-block must be complete so its
last interface row is a real row, not padding).
"""
from __future__ import annotations

from .errors import ValidationError


def split_rows(n: int, world: int, m: int) -> list[int]:
    if world < 1 or n < 1:
        raise ValidationError("need n >= 1 and world >= 1")
    if world == 1:
        return [n]
    q = max(m, (n // world) // m * m)
    last = n - q * (world - 1)
    if last < 1:
        raise ValidationError(f"n = {n} too small for {world} ranks with m = {m}")
    return [q] * (world - 1) + [last]


def row_offset(n: int, world: int, m: int, rank: int) -> int:
    return sum(split_rows(n, world, m)[:rank])


class DistributedSolver:
    """Collective row-sharded solve over an initialised torch.distributed group
    (backend nccl on GPUs; every rank calls `solve`)."""

    def __init__(self, solver, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.solver = solver
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        dev = device if device is not None else torch.device("cuda", solver.device)
        self.iface = torch.zeros(8, dtype=torch.float64, device=dev)
        self.iface_all = torch.zeros(8 * self.world, dtype=torch.float64, device=dev)

    def _all_gather(self):
        if self.iface.is_cuda and self.dist.get_backend(self.group) != "nccl":
            # host-staged exchange for backends without CUDA collectives (tests)
            h, hall = self.iface.cpu(), self.iface_all.cpu()
            self.dist.all_gather_into_tensor(hall, h, group=self.group)
            self.iface_all.copy_(hall)
        else:
            self.dist.all_gather_into_tensor(self.iface_all, self.iface, group=self.group)

    def solve_host(self, a, b, c, d, x, m: int = 10, stream=None):
        """End-to-end collective solve from this rank's host rows (page-locked
        numpy arrays, e.g. `pinned_empty`): H2D of a, b, c, d into device
        staging owned by this object, the row-sharded solve, D2H of x.
        Synchronous; returns x."""
        import numpy as np
        import torch

        n = int(len(b))
        for t in (a, b, c, d, x):
            if not (isinstance(t, np.ndarray) and t.dtype == b.dtype and t.dtype in (np.float64, np.float32)
                    and t.flags.c_contiguous and len(t) == n):
                raise ValidationError("host arrays must be contiguous float64/float32 of equal length")
        dev = self.iface.device
        tdt = torch.float64 if b.dtype == np.float64 else torch.float32
        if getattr(self, "_stage", None) is None or self._stage.shape[1] < n or self._stage.dtype != tdt:
            self._stage = torch.empty((5, n), dtype=tdt, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        da, db, dc, dd, dx = (self._stage[k, :n] for k in range(5))
        with torch.cuda.stream(st):
            for dst, src in ((da, a), (db, b), (dc, c), (dd, d)):
                dst.copy_(torch.from_numpy(src), non_blocking=True)
            self.solve(da, db, dc, dd, dx, m=m, stream=st)
            xh = torch.from_numpy(x)
            xh.copy_(dx, non_blocking=True)
        st.synchronize()
        self.solver.check()
        return x

    def solve(self, a, b, c, d, x, m: int = 10, stream=None):
        if self.iface.dtype != b.dtype:  # FP32 solve: interface equations in FP32
            self.iface = self.iface.to(b.dtype)
            self.iface_all = self.iface_all.to(b.dtype)
        self.solver.dist_reduce(a, b, c, d, m, self.rank, self.world, self.iface, stream=stream)
        self._all_gather()
        self.solver.dist_solve(a, b, c, d, x, m, self.rank, self.world, self.iface_all, stream=stream)
        return x
