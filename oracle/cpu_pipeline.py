"""CPU port of the reference's per-batch lookup pipeline — the CPU baseline
(TEST/BENCH INFRASTRUCTURE ONLY; bench.py's cpu_baseline and --impl
reference legs).

Restates Ranker.execute_batch with the cache off (ranker.py:218-301 fan-out,
305-328 server handler, 364-415 combine) on host numpy tables, one table per
server (table-wise placement, table t on server t): per (lookup, feature)
the indices are grouped by server (routing.py:117-148), planned against the
pushdown threshold (pooling.py:88-100), pushed-down groups are gathered and
summed row by row in f64 (store.py:184-193, pooling.py:60-71) and the ranker
combines partials and raw rows (pooling.py:103-123). The virtual transport's
event loop is not modelled (it only adds cost on the reference side).
"""

from __future__ import annotations

import os
import time

import numpy as np

from .restate import rows_of


class RefPipelinePort:
    def __init__(self, seed: int, table_rows, dim: int, row_cap: int | None = None, threshold: int | None = 2):
        """Materialise host tables (rows capped at `row_cap`: a row-reduced
        replica, indices are taken modulo the cap; per-row cost is independent
        of table size)."""
        self.dim = dim
        self.threshold = threshold
        self.tables = []
        self.rows = []
        for t, n in enumerate(table_rows):
            m = n if row_cap is None else min(n, row_cap)
            self.rows.append(m)
            self.tables.append(rows_of(seed, t, dim, np.arange(m, dtype=np.int64)))

    def _partial_pool(self, t, idx):
        rows = self.tables[t][idx]                      # lookup_rows: fancy-index gather
        acc = np.zeros(self.dim, dtype=np.float64)      # sum_rows_f64: per-row f64 loop
        for r in rows:
            acc += r
        return acc.astype(np.float32), len(idx)

    def run(self, host_batch, samples):
        """Pool bags (s, f) for s in `samples`; returns dict bag -> f32 vector."""
        B = host_batch.batch_size
        out = {}
        thr = self.threshold
        for s in samples:
            for f, t in enumerate(host_batch.feature_tables):
                b = f * B + s
                idx = host_batch.indices[host_batch.offsets[b]:host_batch.offsets[b + 1]].astype(np.int64)
                idx %= self.rows[t]
                # group_by_server: one server per table -> one group, positions 0..L-1
                partials, raw = [], []
                if thr is not None and len(idx) >= thr:
                    partials.append(self._partial_pool(t, idx))
                else:
                    raw = list(self.tables[t][idx])
                vecs = [p[0] for p in partials] + raw
                acc = np.zeros(self.dim, dtype=np.float64)
                for v in vecs:
                    acc += v
                if host_batch.feature_ops[f] == "mean":
                    acc = acc / (sum(p[1] for p in partials) + len(raw))
                out[b] = acc.astype(np.float32)
        return out


_STATE = None


def _worker(samples):
    port, hb = _STATE
    t0 = time.perf_counter()
    port.run(hb, samples)
    return time.perf_counter() - t0, len(samples) * len(hb.feature_tables)


class ParallelPort:
    """Persistent forked worker pool over disjoint sample slices (BASELINE.md
    CPU-baseline plan: os.cpu_count() processes, embarrassingly parallel)."""

    def __init__(self, port, hb, procs: int | None = None):
        import multiprocessing as mp
        global _STATE
        _STATE = (port, hb)
        self.procs = procs or os.cpu_count() or 1
        self.hb = hb
        self.pool = mp.get_context("fork").Pool(self.procs)

    def step(self, samples_per_proc: int, offset: int = 0):
        """One step: every process pools its own slice; returns (bags/s, wall s)."""
        B = self.hb.batch_size
        slices = [[(offset + p * samples_per_proc + i) % B for i in range(samples_per_proc)]
                  for p in range(self.procs)]
        t0 = time.perf_counter()
        res = self.pool.map(_worker, slices)
        wall = time.perf_counter() - t0
        return sum(r[1] for r in res) / wall, wall

    def close(self):
        self.pool.close()
        self.pool.join()


def time_parallel(port, hb, samples_per_proc: int, procs: int | None = None):
    """One-shot variant of ParallelPort.step (includes the fork)."""
    pp = ParallelPort(port, hb, procs)
    try:
        r, wall = pp.step(samples_per_proc)
    finally:
        pp.close()
    return r, pp.procs, wall
