"""CPU oracle for the embedding-lookup hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy / plain Python, the algorithm of the
reference `embserve` package (FlexEMR, arXiv 2410.12794) for the hot path
named in BASELINE.json: table content PRF, gather + fp64 pooling, combine,
range routing, per-batch dedup, the adaptive hot-row cache (canonical order)
and the batch pipeline's counters. Every function cites the reference
file:line it follows (paths relative to /root/reference/pkg/src/embserve).

Parity pinning: the restatement is checked against golden vectors produced
by the reference itself (tests/golden/make_golden.py imports the reference
in the build container; the committed .npz/.json fixtures travel with the
repo). See tests/test_oracle_golden.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or
the CPU baseline. The product package (paper_2410_12794_b200) never imports
it and has no CPU fallback.
"""

from .restate import *  # noqa: F401,F403
