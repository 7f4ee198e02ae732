#!/usr/bin/env python
"""Small solves through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) -- a verification tool, not
product code.  Exits non-zero if a result misses the parity bars."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import oracle
    from paper_2501_05938_b200 import PartitionSolver, pinned_empty
    from paper_2501_05938_b200.solver import PM_OPT_BATCH_CLUSTER

    def check(x, a, b, c, d, tol=1e-10):
        xr = oracle.thomas(a, b, c, d)
        e = oracle.rel_err(np.ascontiguousarray(x, np.float64), xr)
        assert e <= tol, e

    s = PartitionSolver(0)
    if "--no-pdl" in sys.argv:
        from paper_2501_05938_b200.solver import PM_OPT_PDL

        s.set_option(PM_OPT_PDL, 0)
    st = torch.cuda.Stream()
    for n, m in ((70_001, 10), (200_003, 10), (9_999, 7), (3_000, 16)):  # 200_003: fused upper levels
        a, b, c, d = oracle.generate(n, n)
        t = [torch.from_numpy(v).cuda() for v in (a, b, c, d)]
        with torch.cuda.stream(st):
            x = s.solve_device(*t, m=m, stream=st)
        s.check()
        check(x.cpu().numpy(), a, b, c, d)
        x32 = s.solve_device(*[v.float() for v in t], m=m)
        s.check()
        check(x32.cpu().numpy(), *(v.astype(np.float32).astype(np.float64) for v in (a, b, c, d)), tol=1e-5)
    n = 200_001
    a, b, c, d = oracle.generate(n, 1)
    host = [pinned_empty(n) for _ in range(5)]
    for h, v in zip(host, (a, b, c, d)):
        h[:] = v
    check(s.solve_host(*host[:4], m=10, num_streams=4, out=host[4]), a, b, c, d)
    nps, batch = 4_000, 6
    a, b, c, d = oracle.generate(nps * batch, 2)
    t = [torch.from_numpy(v).cuda() for v in (a, b, c, d)]
    from paper_2501_05938_b200.solver import PM_OPT_BATCH_WARPS, PM_OPT_MAX_CTAS, PM_OPT_UPPER_FUSED

    for cl in (0, 1, 2):  # level kernels, cluster kernel, tile-stream kernel (small grid: many rounds)
        s.set_option(PM_OPT_BATCH_CLUSTER, cl)
        s.set_option(PM_OPT_MAX_CTAS, 4 if cl == 2 else 0)
        s.set_option(PM_OPT_BATCH_WARPS, 4 if cl == 2 else 0)
        xb = s.solve_batch_device(*t, n_per_system=nps, m=10).cpu().numpy()
        s.check()
        for k in range(batch):
            sl = slice(k * nps, (k + 1) * nps)
            sa, sc = a[sl].copy(), c[sl].copy()
            sa[0] = 0.0
            sc[-1] = 0.0
            check(xb[sl], sa, b[sl].copy(), sc, d[sl].copy())
        if cl == 2:
            assert s.last_batch_plan()["kernel"] == "stream", s.last_batch_plan()
    s.set_option(PM_OPT_BATCH_CLUSTER, 0)
    s.set_option(PM_OPT_MAX_CTAS, 0)
    s.set_option(PM_OPT_BATCH_WARPS, 0)
    # row-sharded, two virtual ranks with the P2P exchange; then the fused
    # upper levels for ranks (PM_OPT_UPPER_FUSED = 2) at a size where they apply
    run_p2p(s, 50_000, 3)
    s.set_option(PM_OPT_UPPER_FUSED, 2)
    run_p2p(s, 2 * 409_600, 4)
    s.set_option(PM_OPT_UPPER_FUSED, 1)
    s.close()
    print("sanitize driver ok")


def run_p2p(s, n, seed):
    import torch

    import oracle
    from paper_2501_05938_b200 import PartitionSolver

    def check(x, a, b, c, d, tol=1e-10):
        e = oracle.rel_err(np.ascontiguousarray(x, np.float64), oracle.thomas(a, b, c, d))
        assert e <= tol, e

    world = 2
    a, b, c, d = oracle.generate(n, seed)
    a, b, c, d = oracle.generate(n, 3)
    other = PartitionSolver(0)
    from paper_2501_05938_b200.solver import PM_OPT_UPPER_FUSED

    other.set_option(PM_OPT_UPPER_FUSED, 2)
    hs = [s, other]
    bufs = [h.dist_exchange_alloc(world) for h in hs]
    for r, h in enumerate(hs):
        h.dist_set_peers(bufs, r)
    half = n // 2
    rows = [half, n - half]
    loc = [[torch.from_numpy(v[r * half:r * half + rows[r]].copy()).cuda() for v in (a, b, c, d)]
           for r in range(world)]
    for r in range(world):
        hs[r].dist_reduce_p2p(*loc[r], m=10)
    xs = []
    for r in range(world):
        x = torch.empty(rows[r], dtype=torch.float64, device="cuda")
        hs[r].dist_solve_p2p(*loc[r], x, m=10)
        xs.append(x)
    for h in hs:
        h.check()
    check(torch.cat(xs).cpu().numpy(), a, b, c, d)
    other.close()


if __name__ == "__main__":
    main()
