"""CPU oracle for the BLaST hot path (TEST INFRASTRUCTURE ONLY).

A numpy restatement of the reference package's hot path (pkg/src/blocksparse
bcsc.py / kernels.py / mlp.py / pruner.py / bench.py:random_bcsc), used solely as
the checker: by tests/, by __graft_entry__.smoke() and by bench.py's
``cpu_baseline`` / ``--impl reference`` leg. The product (paper_2507_03117_b200)
never imports it. It is pinned against golden vectors produced by running the
real reference package (tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""
from .ref_numpy import *  # noqa: F401,F403
