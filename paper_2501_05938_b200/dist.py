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

from .errors import CudaRuntimeError, ValidationError


def split_rows(n: int, world: int, m: int) -> list[int]:
    if world < 1 or n < 1:
        raise ValidationError("need n >= 1 and world >= 1")
    if world == 1:
        return [n]
    # non-last ranks: whole level-0 tiles in groups of 4 (128*m rows) when the
    # share allows, so level 1 holds whole 8-row blocks and the rank's upper
    # levels run fused (two launches); else a multiple of m
    unit = 128 * m if n // world >= 128 * m else m
    q = max(m, (n // world) // unit * unit)
    last = n - q * (world - 1)
    if last < 1:
        raise ValidationError(f"n = {n} too small for {world} ranks with m = {m}")
    return [q] * (world - 1) + [last]


def row_offset(n: int, world: int, m: int, rank: int) -> int:
    return sum(split_rows(n, world, m)[:rank])


class DistributedSolver:
    """Collective row-sharded solve over an initialised torch.distributed group
    (every rank calls `solve`).

    exchange="p2p" (default when it works): the interface equations travel
    through peer memory -- every rank's exchange buffer is mapped into every
    other rank with CUDA IPC (NVLink), pm_dist_reduce_p2p publishes this
    rank's 64 bytes into every peer and pm_dist_solve_p2p waits on the peers'
    epoch flags inside the solve kernel: no collective call and no host sync
    on the data path.  torch.distributed only carries the one-time handle
    exchange (and the self-test that validates the mapping).
    exchange="collective": all_gather_into_tensor of the 8 doubles per rank
    (NCCL over NVLink; gloo stages through the host).
    """

    def __init__(self, solver, group=None, device=None, exchange: str = "auto"):
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
        self._opened = []
        self.last_launches = 0
        self.exchange = "collective"
        if exchange in ("auto", "p2p"):
            if self._setup_p2p():
                self.exchange = "p2p"
            elif exchange == "p2p":
                raise CudaRuntimeError("P2P interface exchange unavailable on this group")

    def _agree(self, ok: bool) -> bool:
        """All ranks agree on a flag (logical AND over the group)."""
        import torch

        dev = self.iface.device if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return bool(t.item())

    def _setup_p2p(self) -> bool:
        """Map every rank's exchange buffer (CUDA IPC) and register them, then
        validate the mapping with one exchange.  Every rank takes part in the
        same collectives whatever fails locally, and all ranks agree on the
        outcome, so a partial failure falls back to the all-gather everywhere
        instead of deadlocking."""
        import torch

        from .solver import ipc_get_handle, ipc_open_handle

        ok = True
        try:
            own = self.solver.dist_exchange_alloc(self.world)
            raw = ipc_get_handle(own)
        except Exception:
            ok, own, raw = False, 0, bytes(64)
        h = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
        if self.dist.get_backend(self.group) == "nccl":
            hs = [torch.empty(64, dtype=torch.uint8, device=self.iface.device) for _ in range(self.world)]
            self.dist.all_gather(hs, h.to(self.iface.device), group=self.group)
            hs = [t.cpu() for t in hs]
        else:
            hs = [torch.empty(64, dtype=torch.uint8) for _ in range(self.world)]
            self.dist.all_gather(hs, h, group=self.group)
        if ok:
            try:
                ptrs = []
                for k, hk in enumerate(hs):
                    if k == self.rank:
                        ptrs.append(own)
                    else:
                        p = ipc_open_handle(bytes(hk.numpy().tobytes()))
                        self._opened.append(p)
                        ptrs.append(p)
                self.solver.dist_set_peers(ptrs, self.rank)
                torch.cuda.synchronize()
            except Exception:
                ok = False
        # every buffer cleared (set_peers) before anyone publishes
        if not self._agree(ok):
            self.close()
            return False
        try:  # self-test: one exchange of tiny systems through the mapping
            n = 40
            t = [torch.full((n,), v, dtype=torch.float64, device=self.iface.device)
                 for v in (0.5, 4.0, 0.5, 1.0)]
            x = torch.empty(n, dtype=torch.float64, device=self.iface.device)
            self.solver.dist_reduce_p2p(*t, m=10)
            self.solver.dist_solve_p2p(*t, x, m=10)
            self.solver.check()
        except Exception:
            ok = False
        if not self._agree(ok):
            self.close()
            return False
        return True

    def _all_gather(self):
        if self.iface.is_cuda and self.dist.get_backend(self.group) != "nccl":
            # host-staged exchange for backends without CUDA collectives (tests)
            h, hall = self.iface.cpu(), self.iface_all.cpu()
            self.dist.all_gather_into_tensor(hall, h, group=self.group)
            self.iface_all.copy_(hall)
        else:
            self.dist.all_gather_into_tensor(self.iface_all, self.iface, group=self.group)

    def close(self):
        from .solver import ipc_close_handle

        for p in self._opened:
            ipc_close_handle(p)
        self._opened = []

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
        if self.exchange == "p2p":
            self.solver.dist_reduce_p2p(a, b, c, d, m, stream=stream)
            k = getattr(self.solver, "last_launch_count", 0)
            self.solver.dist_solve_p2p(a, b, c, d, x, m, stream=stream)
            self.last_launches = k + getattr(self.solver, "last_launch_count", 0)
            return x
        if self.iface.dtype != b.dtype:  # FP32 solve: interface equations in FP32
            self.iface = self.iface.to(b.dtype)
            self.iface_all = self.iface_all.to(b.dtype)
        import contextlib

        import torch

        # the exchange runs on the solve's stream: NCCL (and gloo's .cpu()) order
        # against the current stream, which must be the one dist_reduce wrote
        # iface on and dist_solve reads iface_all on
        if isinstance(stream, int):  # raw cudaStream_t
            stream = torch.cuda.ExternalStream(stream, device=self.iface.device)
        ctx = (torch.cuda.stream(stream) if stream is not None and self.iface.is_cuda
               else contextlib.nullcontext())
        with ctx:
            self.solver.dist_reduce(a, b, c, d, m, self.rank, self.world, self.iface, stream=stream)
            k = getattr(self.solver, "last_launch_count", 0)
            self._all_gather()
            self.solver.dist_solve(a, b, c, d, x, m, self.rank, self.world, self.iface_all, stream=stream)
        # the solver's own kernels (the all-gather's NCCL kernel is not counted)
        self.last_launches = k + getattr(self.solver, "last_launch_count", 0)
        return x
