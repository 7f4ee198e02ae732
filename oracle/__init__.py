"""CPU oracle for the partition-method solver -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
as the timed CPU baseline.  The product package ``paper_2501_05938_b200``
never imports it.  See ``oracle/tridiag_oracle.c`` for what it restates and
``tests/test_oracle.py`` for how it is pinned (LAPACK dgtsv, golden fixtures,
and the reference's own timing-model header compiled into ``oracle/_ref``).
"""
from .oracle import *  # noqa: F401,F403
