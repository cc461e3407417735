"""Synthetic lookup workloads (embserve/workload.py:111-126 ZipfSampler
semantics) and the BASELINE.json configurations — numpy only.

Inputs are generated once on the host and consumed identically by the GPU
path, the CPU oracle and the reference arm. This module has
no dependency on the product package, so the reference arm of bench.py
(`--impl reference`) can build the same batches without loading
libflexemb.so; paper_2410_12794_b200.workload re-exports it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# Criteo-Kaggle per-feature cardinalities (26 categorical features)
CRITEO_KAGGLE_ROWS = (1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194, 27,
                      14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572)


class ZipfSampler:
    """Exact inverse-CDF Zipf(alpha) over n row ids, row r has probability
    (r+1)^-alpha / H_n(alpha) (workload.py:111-126)."""

    def __init__(self, n: int, alpha: float):
        if n < 1:
            raise ValueError("zipf sampler needs n >= 1")
        self.n = n
        self.alpha = alpha
        w = np.arange(1, n + 1, dtype=np.float64) ** (-alpha)
        self.pmf = w / w.sum()
        self.cdf = np.cumsum(self.pmf)

    def sample(self, rng: np.random.Generator, count: int) -> np.ndarray:
        return np.searchsorted(self.cdf, rng.random(count), side="right")

    def from_uniform(self, u: np.ndarray) -> np.ndarray:
        """Same mapping for pre-drawn uniforms; the (prob ~1e-14) draw past
        cdf[-1] is clamped to n-1."""
        r = np.searchsorted(self.cdf, u, side="right")
        np.minimum(r, self.n - 1, out=r)
        return r


@dataclass
class HostBatch:
    """Host CSR batch, table-major bags (bag = f*B + s)."""

    indices: np.ndarray   # int32 [nnz]
    offsets: np.ndarray   # int64 [F*B + 1]
    feature_tables: tuple
    feature_ops: tuple
    batch_size: int

    @property
    def nnz(self) -> int:
        return int(self.offsets[-1])

    def to_lists(self):
        """Reference-shaped lookups: list (per sample) of (table, op, indices)."""
        B, F = self.batch_size, len(self.feature_tables)
        out = []
        for s in range(B):
            feats = []
            for f in range(F):
                b = f * B + s
                feats.append((self.feature_tables[f], self.feature_ops[f],
                              self.indices[self.offsets[b]:self.offsets[b + 1]].tolist()))
            out.append(feats)
        return out


class DlrmBatchGen:
    """Per-batch generator: one feature per table, Zipf(alpha) rows.

    RNG order per batch: bag lengths (if ragged) as one (B, F) draw, then
    all uniforms in (sample, feature, position) order; each table maps its
    uniforms through its own inverse CDF. `permute` applies a fixed bijective
    row permutation r -> (a*r + c) mod n per table (breaks the row-id =
    popularity-rank locality for row-wise sharding, SURVEY §7 hard part 4)."""

    def __init__(self, table_rows, alpha: float, batch_size: int, pooling, seed: int = 0,
                 ops=None, tables=None, permute: bool = False):
        self.table_rows = tuple(int(r) for r in table_rows)
        self.tables = tuple(tables) if tables is not None else tuple(range(len(self.table_rows)))
        self.ops = tuple(ops) if ops is not None else tuple("sum" for _ in self.tables)
        self.B = batch_size
        self.pooling = pooling if isinstance(pooling, tuple) else (int(pooling), int(pooling))
        self.rng = np.random.default_rng(seed)
        self.samplers = {}
        self.alpha = alpha
        self.permute = permute
        for n in set(self.table_rows):
            self.samplers[n] = ZipfSampler(n, alpha)

    def _perm(self, rows: np.ndarray, n: int, t: int) -> np.ndarray:
        a = 2654435761 % n if n > 1 else 1
        while np.gcd(a, n) != 1:
            a += 1
        c = (t * 40503) % n
        return ((rows.astype(np.int64) * a + c) % n).astype(rows.dtype)

    def next(self) -> HostBatch:
        B, F = self.B, len(self.tables)
        lo, hi = self.pooling
        if hi > lo:
            lens = self.rng.integers(lo, hi + 1, size=(B, F))
        else:
            lens = np.full((B, F), lo, dtype=np.int64)
        u = self.rng.random(int(lens.sum()))
        # u is in sample-major (s, f, k) order; regroup table-major
        sm_off = np.concatenate([[0], np.cumsum(lens.reshape(-1))])
        lens_tm = lens.T.reshape(-1)                       # bag = f*B + s
        offsets = np.concatenate([[0], np.cumsum(lens_tm)]).astype(np.int64)
        indices = np.empty(int(offsets[-1]), dtype=np.int32)
        for f in range(F):
            n = self.table_rows[f]
            starts = sm_off[np.arange(B) * F + f]
            ln = lens[:, f]
            pos = np.repeat(starts, ln) + (np.arange(ln.sum()) - np.repeat(np.cumsum(ln) - ln, ln))
            rows = self.samplers[n].from_uniform(u[pos]).astype(np.int32)
            if self.permute:
                rows = self._perm(rows, n, self.tables[f])
            indices[offsets[f * B]:offsets[(f + 1) * B]] = rows
        return HostBatch(indices, offsets, self.tables, self.ops, B)


# ---- BASELINE.json configurations ------------------------------------------------

CONFIGS = {
    # configs[0]: the reference CPU pipeline case
    "cfg1": dict(name="ref-cpu-pipeline-8x100Kx64", table_rows=(100_000,) * 8, dim=64, batch=512, pooling=20,
                 alpha=1.05),
    # configs[1]: Criteo-Kaggle-shaped, single B200 (the bench workload)
    "cfg2": dict(name="criteo-kaggle-26x128", table_rows=CRITEO_KAGGLE_ROWS, dim=128, batch=4096, pooling=(1, 40),
                 alpha=1.05),
    "cfg3": dict(name="hot-cache-32x10Mx128", table_rows=(10_000_000,) * 32, dim=128, batch=4096, pooling=20,
                 alpha=1.0),
    "cfg4": dict(name="dlrm-rm2-100x10Mx128-tablewise", table_rows=(10_000_000,) * 100, dim=128, batch=4096,
                 pooling=20, alpha=1.05),
    "cfg5": dict(name="fanout-200x1Mx128-rowwise", table_rows=(1_000_000,) * 200, dim=128, batch=4096,
                 pooling=100, alpha=1.0, permute=True),
    # cfg4 row-reduced variant for the 1->2->4->8 curve
    "cfg4r": dict(name="dlrm-rm2-100x1Mx128-tablewise-rowreduced", table_rows=(1_000_000,) * 100, dim=128,
                  batch=4096, pooling=20, alpha=1.05),
}
