"""Python host-side mirror of the solver's C ABI (include/pm_tridiag.h).

Same entry points, argument meaning and error behaviour as the C ABI:
status 1 -> ValidationError, 2 -> ComputationError, 3 -> CudaRuntimeError
(the streamtune taxonomy, /root/reference/proj/include/streamtune/
errors.hpp:9-21).  Arrays are float64 numpy arrays (host path) or float64
CUDA torch tensors (device paths); `a[0]` and `c[n-1]` are ignored.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .errors import ComputationError, CudaRuntimeError, ValidationError, raise_for

PM_OPT_STAGES = 1
PM_OPT_STREAM_MODE = 2
PM_OPT_REVERSE_SOLVE = 3
PM_OPT_MAX_CTAS = 4
PM_OPT_TIMINGS = 5
PM_OPT_KERNEL_TIMES = 6
PM_OPT_WARP_TILES = 7
PM_OPT_SOLVE_STAGES = 8
PM_OPT_WARPS_PER_CTA = 9
PM_OPT_CHAIN = 10
PM_OPT_UPPER_M = 11
PM_OPT_ROOT_M = 12
PM_OPT_PDL = 13
PM_OPT_BATCH_CLUSTER = 14
PM_OPT_BATCH_L2_MB = 15
PM_OPT_BATCH_CLUSTER_SIZE = 16
PM_OPT_BATCH_WARPS = 17
PM_OPT_BATCH_STAGES = 18
PM_OPT_BATCH_LAG = 25
PM_OPT_BATCH_DISCARD = 26
PM_OPT_BATCH_STATS = 27
PM_OPT_PAIR_TILES = 19
PM_OPT_UPPER_CTA_M = 20
PM_OPT_UPPER_CTA_P = 21
PM_OPT_GRAPHS = 22
PM_OPT_PAIR_STAGES = 23
PM_OPT_UPPER_FUSED = 24
PM_MAX_M = 128


@dataclass
class StageTimings:
    """streamtune::StageTimings (timing_model.hpp:77-85), milliseconds."""
    slae_size: int = 0
    t1_h2d: float = 0.0
    t1_comp: float = 0.0
    t1_d2h: float = 0.0
    t2_comp: float = 0.0
    t3_h2d: float = 0.0
    t3_comp: float = 0.0
    t3_d2h: float = 0.0


def _check_host(*arrs, dtype=np.float64):
    for x in arrs:
        if not isinstance(x, np.ndarray) or x.dtype != dtype or not x.flags.c_contiguous:
            raise ValidationError(f"host arrays must be C-contiguous {np.dtype(dtype).name} numpy arrays")


def _suffix(dtype) -> str:
    """C ABI precision suffix of a torch / numpy dtype: FP64 (the north_star
    solver) or FP32 (the paper's FP32 experiments)."""
    name = str(dtype).replace("torch.", "")
    if name == "float64":
        return "f64"
    if name == "float32":
        return "f32"
    raise ValidationError("arrays must be float64 or float32")


def _dev_ptr(t, n: Optional[int] = None, dtype=None, device: Optional[int] = None) -> int:
    import torch

    dtype = dtype if dtype is not None else torch.float64
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or not t.is_cuda:
        raise ValidationError(f"device arrays must be {str(dtype).replace('torch.', '')} CUDA tensors")
    if not t.is_contiguous():
        raise ValidationError("device arrays must be contiguous")
    if n is not None and t.numel() < n:
        raise ValidationError("device array shorter than n")
    if device is not None and t.device.index != device:
        raise ValidationError(f"device array on cuda:{t.device.index}, the solver's handle is on cuda:{device}")
    return t.data_ptr()


def _stream_handle(stream) -> int:
    import torch

    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class PartitionSolver:
    """One handle per GPU / host thread (pm_create .. pm_destroy)."""

    def __init__(self, device: int = 0, stages: Optional[int] = None, stream_mode: Optional[int] = None,
                 reverse_solve: Optional[bool] = None, timings: bool = False):
        self._L = _lib.load()
        h = C.c_void_p()
        st = self._L.pm_create(C.byref(h), int(device))
        if st != 0:
            raise CudaRuntimeError(f"pm_create failed on device {device} (status {st})")
        self._h = h
        self.device = device
        if stages is not None:
            self.set_option(PM_OPT_STAGES, stages)
        if stream_mode is not None:
            self.set_option(PM_OPT_STREAM_MODE, stream_mode)
        if reverse_solve is not None:
            self.set_option(PM_OPT_REVERSE_SOLVE, int(reverse_solve))
        self.set_option(PM_OPT_TIMINGS, int(timings))

    # -- plumbing -------------------------------------------------------------
    def _ptr(self, t, n: Optional[int] = None, dtype=None) -> int:
        """Device pointer of `t`, validated to live on this handle's device."""
        return _dev_ptr(t, n, dtype, int(self.device))

    def _ok(self, st: int):
        if st != 0:
            raise_for(st, self._L.pm_last_error(self._h).decode(errors="replace"))

    def close(self):
        if getattr(self, "_h", None):
            self._L.pm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_option(self, option: int, value: int):
        self._ok(self._L.pm_set_option(self._h, option, int(value)))

    @property
    def last_launch_count(self) -> int:
        return int(self._L.pm_last_launch_count(self._h))

    def last_batch_plan(self) -> dict:
        """Batch-kernel configuration of the last batch solve: "kernel" is
        "level", "cluster" (cluster, warps, stages, kmax, ntiles, clusters) or
        "stream" (stream = {warps, stages, lag, ring, ctas, nw, tps})."""
        out = (C.c_int32 * 6)()
        self._L.pm_last_batch_plan(self._h, out)
        d = dict(zip(("cluster", "warps", "stages", "kmax", "ntiles", "clusters"), list(out)))
        sp = (C.c_int32 * 8)()
        self._L.pm_last_stream_plan(self._h, sp)
        d["stream"] = dict(zip(("warps", "stages", "lag", "ring", "ctas", "nw", "tps"), list(sp)[1:])) \
            if sp[0] else None
        d["kernel"] = "stream" if sp[0] else ("cluster" if d["cluster"] else "level")
        return d

    def batch_stream_stats(self) -> dict:
        """Diagnostics of the last tile-stream launch (PM_OPT_BATCH_STATS)."""
        out = (C.c_uint64 * 15)()
        self._ok(self._L.pm_batch_stream_stats(self._h, out))
        keys = ("cflag_wait_cyc", "cflag_waits", "mbox_wait_cyc", "stage_wait_cyc", "ctl_iters", "ctl_idle",
                "stage2_cyc", "stage2_n", "publish_cyc", "compute_cyc", "control_cyc", "a_jobs", "c_jobs", "queue_ns",
                "s2_latency_ns")
        return dict(zip(keys, [int(v) for v in out]))

    def batch_stream_timeline(self, batch: int):
        """Per-system globaltimer stamps of the last tile-stream launch with
        PM_OPT_BATCH_STATS: a [5, batch] uint64 array (first Stage-1 start,
        last Stage-1 end, Stage-1 count complete, Stage-2 flag, first Stage-3
        wait start)."""
        import numpy as np

        out = np.zeros(5 * batch + 8 * 2400 * 4 + 1200 * 2 + 4096 * 12, dtype=np.uint64)
        self._ok(self._L.pm_batch_stream_timeline(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                  C.c_int64(out.size)))
        return out[:5 * batch].reshape(5, batch)

    def batch_stream_traces(self, batch: int):
        """Job traces of 8 sample compute warps ([8, 2400, 4]: code, start,
        stage ready, end) and the control-warp iterations of CTA 0 ([1200, 2])."""
        import numpy as np

        out = np.zeros(5 * batch + 8 * 2400 * 4 + 1200 * 2 + 4096 * 12, dtype=np.uint64)
        self._ok(self._L.pm_batch_stream_timeline(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                  C.c_int64(out.size)))
        o = 5 * batch
        o2 = o + 8 * 2400 * 4 + 1200 * 2
        return (out[o:o + 8 * 2400 * 4].reshape(8, 2400, 4), out[o + 8 * 2400 * 4:o2].reshape(1200, 2),
                out[o2:].reshape(4096, 12))

    def last_plan(self) -> list[int]:
        buf = (C.c_int64 * 16)()
        k = self._L.pm_last_plan(self._h, buf, 16)
        return [int(buf[i]) for i in range(min(k, 16))]

    # -- solves -----------------------------------------------------------------
    def solve_host(self, a, b, c, d, m: int = 10, num_streams: int = 0, out=None) -> np.ndarray:
        """pm_solve_host_f64 / _f32 (by the arrays' dtype): host arrays in, x out
        (copies overlap compute when the arrays are page-locked, e.g.
        `pinned_empty`)."""
        dt = b.dtype if isinstance(b, np.ndarray) else np.float64
        sfx = _suffix(dt)
        _check_host(a, b, c, d, dtype=dt)
        n = b.shape[0]
        if not (a.shape[0] == c.shape[0] == d.shape[0] == n):
            raise ValidationError("a, b, c, d must have the same length")
        x = out if out is not None else np.empty(n, dt)
        _check_host(x, dtype=dt)
        fn = getattr(self._L, "pm_solve_host_" + sfx)
        self._ok(fn(self._h, a.ctypes.data, b.ctypes.data, c.ctypes.data, d.ctypes.data, x.ctypes.data, n,
                    m, num_streams))
        return x

    def solve_device(self, a, b, c, d, m: int = 10, out=None, stream=None, n: Optional[int] = None):
        """pm_solve_device_f64 / _f32 by b's dtype (asynchronous; `check()`
        reports pivot failures)."""
        import torch

        dt = b.dtype
        fn = getattr(self._L, "pm_solve_device_" + _suffix(dt))
        n = int(b.numel()) if n is None else n
        x = out if out is not None else torch.empty(n, dtype=dt, device=b.device)
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt),
                    self._ptr(x, n, dt), n, m, _stream_handle(stream)))
        return x

    def solve_batch_device(self, a, b, c, d, n_per_system: int, m: int = 10, out=None, stream=None):
        import torch

        dt = b.dtype
        fn = getattr(self._L, "pm_solve_batch_device_" + _suffix(dt))
        n = int(b.numel())
        if n_per_system < 1 or n % n_per_system:
            raise ValidationError("array length must be a multiple of n_per_system")
        x = out if out is not None else torch.empty(n, dtype=dt, device=b.device)
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt),
                    self._ptr(x, n, dt), n_per_system, n // n_per_system, m, _stream_handle(stream)))
        return x

    def solve_batch_host(self, a, b, c, d, n_per_system: int, m: int = 10, depth: int = 0,
                         systems_per_chunk: int = 0, out=None) -> np.ndarray:
        """pm_solve_batch_host_f64 / _f32: a batch from host memory, chunked
        H2D / solve / D2H overlapped on three streams (synchronous)."""
        dt = b.dtype if isinstance(b, np.ndarray) else np.float64
        sfx = _suffix(dt)
        _check_host(a, b, c, d, dtype=dt)
        n = b.shape[0]
        if n_per_system < 1 or n % n_per_system:
            raise ValidationError("array length must be a multiple of n_per_system")
        x = out if out is not None else np.empty(n, dt)
        _check_host(x, dtype=dt)
        fn = getattr(self._L, "pm_solve_batch_host_" + sfx)
        self._ok(fn(self._h, a.ctypes.data, b.ctypes.data, c.ctypes.data, d.ctypes.data, x.ctypes.data,
                    n_per_system, n // n_per_system, m, depth, systems_per_chunk))
        return x

    def check(self):
        """pm_check: synchronise and raise ComputationError on a pivot failure.
        After a flagged device-resident solve it first re-runs that solve with
        classic pivot sweeps (into the same x), so read x after check()."""
        self._ok(self._L.pm_check(self._h))

    def generate_device(self, n: int, seed: int = 42, device=None, stream=None, arrays=None, dtype=None):
        """pm_generate_f64 / _f32 into (new or given) CUDA tensors a, b, c, d."""
        return self.generate_range_device(n, 0, n, seed, device=device, stream=stream, arrays=arrays,
                                          dtype=dtype)

    def generate_range_device(self, n_total: int, row0: int, count: int, seed: int = 42, device=None,
                              stream=None, arrays=None, dtype=None):
        """pm_generate_range_f64 / _f32: rows [row0, row0+count) of the n_total system."""
        import torch

        dev = device if device is not None else torch.device("cuda", self.device)
        if arrays is not None:
            dtype = arrays[1].dtype
        dtype = dtype if dtype is not None else torch.float64
        if arrays is None:
            arrays = [torch.empty(count, dtype=dtype, device=dev) for _ in range(4)]
        fn = getattr(self._L, "pm_generate_range_" + _suffix(dtype))
        self._ok(fn(self._h, *[self._ptr(t, count, dtype) for t in arrays], n_total, row0, count, seed,
                    _stream_handle(stream)))
        return arrays

    def kernel_times(self, max_records: int = 65536):
        """[(mode, level, ms)] recorded while PM_OPT_KERNEL_TIMES is on (synchronises)."""
        modes = (C.c_int32 * max_records)()
        levels = (C.c_int32 * max_records)()
        ms = (C.c_float * max_records)()
        k = self._L.pm_kernel_times(self._h, modes, levels, ms, max_records)
        if k < 0:
            raise CudaRuntimeError(self._L.pm_last_error(self._h).decode())
        return [(int(modes[i]), int(levels[i]), float(ms[i])) for i in range(k)]

    def last_stage_timings(self):
        t = _lib.StageTimingsC()
        total = C.c_double()
        ns = C.c_int32()
        self._ok(self._L.pm_last_stage_timings(self._h, C.byref(t), C.byref(total), C.byref(ns)))
        st = StageTimings(*[getattr(t, f) for f, _ in _lib.StageTimingsC._fields_])
        return st, total.value, ns.value

    # -- row-sharded single system (BASELINE.json config 5) ---------------------
    def dist_reduce(self, a, b, c, d, m: int, rank: int, world: int, iface, stream=None):
        n, dt = int(b.numel()), b.dtype
        fn = getattr(self._L, "pm_dist_reduce_" + _suffix(dt))
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt), n,
                    m, rank, world, self._ptr(iface, 8, dt), _stream_handle(stream)))

    def dist_solve(self, a, b, c, d, x, m: int, rank: int, world: int, iface_all, stream=None):
        n, dt = int(b.numel()), b.dtype
        fn = getattr(self._L, "pm_dist_solve_" + _suffix(dt))
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt),
                    self._ptr(x, n, dt), n, m, rank, world, self._ptr(iface_all, 8 * world, dt),
                    _stream_handle(stream)))

    # -- P2P interface exchange (NVLink peer memory; include/pm_tridiag.h) -------
    def dist_exchange_alloc(self, world: int) -> int:
        """This rank's exchange buffer (device pointer, owned by the handle)."""
        out = C.c_void_p()
        self._ok(self._L.pm_dist_exchange_alloc(self._h, int(world), C.byref(out)))
        return int(out.value)

    def dist_set_peers(self, peer_ptrs, rank: int):
        arr = (C.c_void_p * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
        self._ok(self._L.pm_dist_set_peers(self._h, arr, len(peer_ptrs), int(rank)))

    def dist_reduce_p2p(self, a, b, c, d, m: int, stream=None):
        n, dt = int(b.numel()), b.dtype
        fn = getattr(self._L, "pm_dist_reduce_p2p_" + _suffix(dt))
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt), n,
                    m, _stream_handle(stream)))

    def dist_solve_p2p(self, a, b, c, d, x, m: int, stream=None):
        n, dt = int(b.numel()), b.dtype
        fn = getattr(self._L, "pm_dist_solve_p2p_" + _suffix(dt))
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt),
                    self._ptr(x, n, dt), n, m, _stream_handle(stream)))

    # -- one-call collective solve with the caller's exchange (C ABI) -----------
    def solve_dist(self, a, b, c, d, x, m: int, rank: int, world: int, allgather, stream=None):
        """pm_solve_dist_f64 / _f32: reduce -> allgather(send_ptr, recv_ptr,
        bytes_per_rank, stream_ptr) -> solve, every rank collectively.
        `allgather` is a Python callable returning 0 on success; it runs on
        this thread inside the call (the GIL is released around the C call, so
        ranks may be threads)."""
        n, dt = int(b.numel()), b.dtype
        fn = getattr(self._L, "pm_solve_dist_" + _suffix(dt))

        def tramp(send, recv, nbytes, st, _user):
            try:
                return int(allgather(send, recv, nbytes, st) or 0)
            except Exception:  # never unwind through C
                return 1

        cb = _lib.ALLGATHER_FN(tramp)
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt),
                    self._ptr(x, n, dt), n, m, rank, world, cb, None, _stream_handle(stream)))
        return x

    def solve_dist_nccl(self, a, b, c, d, x, m: int, comm: int, stream=None):
        """pm_solve_dist_nccl_f64 / _f32 on an ncclComm_t (see nccl_comm_init)."""
        n, dt = int(b.numel()), b.dtype
        fn = getattr(self._L, "pm_solve_dist_nccl_" + _suffix(dt))
        self._ok(fn(self._h, self._ptr(a, n, dt), self._ptr(b, n, dt), self._ptr(c, n, dt), self._ptr(d, n, dt),
                    self._ptr(x, n, dt), n, m, C.c_void_p(comm), _stream_handle(stream)))
        return x

    def nccl_get_unique_id(self) -> bytes:
        buf = C.create_string_buffer(128)
        self._ok(self._L.pm_nccl_get_unique_id(self._h, buf))
        return buf.raw

    def nccl_comm_init(self, world: int, uid: bytes, rank: int) -> int:
        comm = C.c_void_p()
        self._ok(self._L.pm_nccl_comm_init(self._h, C.byref(comm), int(world), C.c_char_p(bytes(uid)), int(rank)))
        return int(comm.value)

    def nccl_comm_destroy(self, comm: int):
        self._ok(self._L.pm_nccl_comm_destroy(self._h, C.c_void_p(comm)))

    # -- stream-count model -------------------------------------------------------
    def set_model_bundle(self, bundle: "ModelBundleC"):
        self._ok(self._L.pm_set_model_bundle(self._h, C.byref(bundle)))

    def get_model_bundle(self):
        b = _lib.ModelBundleC()
        self._ok(self._L.pm_get_model_bundle(self._h, C.byref(b)))
        return b


def ipc_get_handle(dptr: int) -> bytes:
    """CUDA IPC handle (64 bytes) of a cudaMalloc'd device pointer."""
    buf = C.create_string_buffer(64)
    if _lib.load().pm_ipc_get_handle(C.c_void_p(dptr), buf) != 0:
        raise CudaRuntimeError("cudaIpcGetMemHandle failed")
    return buf.raw


def ipc_open_handle(handle: bytes) -> int:
    out = C.c_void_p()
    if _lib.load().pm_ipc_open_handle(C.c_char_p(bytes(handle)), C.byref(out)) != 0:
        raise CudaRuntimeError("cudaIpcOpenMemHandle failed")
    return int(out.value)


def ipc_close_handle(dptr: int) -> None:
    _lib.load().pm_ipc_close_handle(C.c_void_p(dptr))


def pinned_empty(n: int, dtype=np.float64) -> np.ndarray:
    """A page-locked host array (torch's pinned allocator), float64 or float32."""
    import torch

    tdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    return torch.empty(n, dtype=tdt, pin_memory=True).numpy()


def recommend_streams(n: int, bundle=None) -> int:
    L = _lib.load()
    r = L.pm_recommend_streams(int(n), C.byref(bundle) if bundle is not None else None)
    if r < 1:
        raise ValidationError("invalid SLAE size or model bundle")
    return int(r)
