"""The reference arm: the UNMODIFIED reference `embserve` package timed on
the host cores (TEST/BENCH INFRASTRUCTURE ONLY — bench.py's cpu_baseline and
`--impl reference` legs; never imported by the product package).

`build()` (__graft_entry__.py) copies /root/reference/pkg/src/embserve into
the untracked oracle/_ref/embserve, which travels to the GPU box with the
snapshot like libflexemb.so (nothing here reads /root/reference at run time).
The arm drives the reference's own public API exactly as its experiment
runner does (`run_pipeline`, bench/experiments.py:132-198): init_store ->
build_routing -> create_connections + assign_mapping_aware (the bench
config's 8 units / 8 engines / 8 connections per peer) -> VirtualTransport
-> AdaptiveCache + CachePolicy + LoadTracker -> Ranker.execute_batch, with
the cfg3 semantics of SURVEY §8(d): pushdown threshold None, sketch
admission, admit_per_batch 64, adaptive_cache on with the memory model
pinned so the budget stays at the configured fraction of all rows.

Tables are row-reduced (the reference materialises every table in host
numpy; cfg3's 164 GB cannot), indices taken modulo the reduced row count;
its per-lookup Python cost does not depend on table size (checked by
`rate_vs_rows`). Multi-core: forked processes each replay their own batch
slices through their own Ranker (replicas, like the survey's `mp` probe).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def available() -> bool:
    return os.path.exists(os.path.join(REF, "embserve", "ranker.py"))


def import_reference():
    """Import embserve from oracle/_ref (never the product package). If the
    name is taken by something else (tests/_ref_alias maps `embserve` to the
    mirror), the reference is loaded anyway and the previous entries are
    restored afterwards for their users."""
    if not available():
        raise ImportError(f"{REF}/embserve is missing: run __graft_entry__.build() in the build container")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    cur = sys.modules.get("embserve")
    if cur is not None and not os.path.abspath(getattr(cur, "__file__", "") or "").startswith(REF):
        saved = {k: v for k, v in sys.modules.items() if k == "embserve" or k.startswith("embserve.")}
        for k in saved:
            del sys.modules[k]
        try:
            import embserve  # noqa: F401
            import embserve.errors  # noqa: F401
            import embserve.pooling  # noqa: F401
            ref = {k: v for k, v in sys.modules.items() if k == "embserve" or k.startswith("embserve.")}
        finally:
            for k in list(sys.modules):
                if k == "embserve" or k.startswith("embserve."):
                    del sys.modules[k]
            sys.modules.update(saved)
        return ref["embserve"]
    import embserve  # noqa: F401
    if not os.path.abspath(embserve.__file__).startswith(REF):
        raise ImportError(f"embserve resolved to {embserve.__file__}, not the copy under {REF}")
    return embserve


class RefRanker:
    """One reference Ranker over row-reduced cfg3-shaped tables."""

    def __init__(self, tables: int, rows: int, dim: int, batch: int, cache_frac: float | None = 0.02,
                 threshold=None, admit: int = 64, seed: int = 0):
        import_reference()
        from embserve.cache import AdaptiveCache, CachePolicy, LoadTracker, MemoryModel
        from embserve.ranker import Ranker, RankerParams
        from embserve.routing import build_routing
        from embserve.store import ShardSpec, TableMeta, init_store
        from embserve.transport.topology import assign_mapping_aware, create_connections
        from embserve.transport.virtual import EventLoop, TransportParams, VirtualTransport

        self.rows, self.dim, self.tables = rows, dim, tables
        metas = [TableMeta(t, rows, dim) for t in range(tables)]
        specs = [ShardSpec(t, 0, rows, 0) for t in range(tables)]
        t0 = time.perf_counter()
        self.dep = init_store(metas, specs, seed)
        self.init_s = time.perf_counter() - t0
        routing = build_routing(metas, specs)
        topo = create_connections(8, peers=self.dep.server_ids, conns_per_peer=8)
        transport = VirtualTransport(EventLoop(), topo, assign_mapping_aware(topo, 8), TransportParams())
        cache = policy = tracker = None
        if cache_frac:
            budget = int(tables * rows * cache_frac) * dim * 4
            cache = AdaptiveCache(budget_bytes=budget, admission="sketch")
            policy = CachePolicy(model=MemoryModel(gpu_capacity_bytes=budget + 1_000 + batch, nn_fixed_bytes=1_000,
                                                   nn_per_sample_bytes=1))
            tracker = LoadTracker(window=16, high_watermark=10 ** 9, low_watermark=0)
        self.ranker = Ranker(self.dep, routing, transport,
                             params=RankerParams(pushdown_threshold=threshold, admit_per_batch=admit,
                                                 keep_results=False),
                             cache=cache, policy=policy, tracker=tracker)
        self._next_id = 0

    def make_batch(self, hb, samples):
        """Reference Batch of samples `samples` of a host CSR batch (table-major
        bags, bag = f*B + s), indices modulo the reduced row count."""
        from embserve.pooling import PoolingOp
        from embserve.requests import Batch, Feature, LookupRequest
        B = hb.batch_size
        lookups = []
        for s in samples:
            feats = []
            for f, t in enumerate(hb.feature_tables):
                b = f * B + s
                idx = (hb.indices[hb.offsets[b]:hb.offsets[b + 1]].astype(np.int64) % self.rows).tolist()
                feats.append(Feature(table_id=t, op=PoolingOp(hb.feature_ops[f]), indices=idx))
            lookups.append(LookupRequest(features=feats))
        self._next_id += 1
        return Batch(batch_id=self._next_id, tick=self._next_id, lookups=lookups)

    def execute(self, batch) -> None:
        # Ranker.execute_batch == run_trace([batch]) + results lookup; results
        # are not kept (keep_results=False, the bench config's setting)
        self.ranker.run_trace([batch])


def _worker(args):
    (tables, rows, dim, B, L, alpha, cache_frac, samples_per_step, steps, warmup, proc, seed) = args
    from flexemb_workload import DlrmBatchGen
    rr = RefRanker(tables, rows, dim, B, cache_frac)
    gen = DlrmBatchGen((rows,) * tables, alpha, B, (L, L), seed=seed + proc)
    hb = gen.next()
    rates = []
    for i in range(warmup + steps):
        if (i * samples_per_step) % B + samples_per_step > B:
            hb = gen.next()
        s0 = (i * samples_per_step) % B
        batch = rr.make_batch(hb, range(s0, s0 + samples_per_step))
        t0 = time.perf_counter()
        rr.execute(batch)
        dt = time.perf_counter() - t0
        if i >= warmup:
            rates.append((samples_per_step * tables, dt))
    return rates, rr.init_s


def run_parallel(procs: int, tables: int, rows: int, dim: int, B: int, L: int, alpha: float, cache_frac: float,
                 samples_per_step: int, steps: int, warmup: int, seed: int = 7):
    """Per step (one `samples_per_step`-lookup batch per process) -> list of
    (bags, seconds) per process. Processes are forked and independent."""
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        res = pool.map(_worker, [(tables, rows, dim, B, L, alpha, cache_frac, samples_per_step, steps, warmup, p,
                                  seed) for p in range(procs)])
    return res


def rate_vs_rows(rows_list=(20_000, 200_000), tables=32, dim=128, B=4096, L=20, alpha=1.0, samples=64, steps=3,
                 warmup=1):
    """Reference bags/s on one core at several row-reduced table sizes
    (evidence that the per-lookup CPU cost does not depend on table size)."""
    out = {}
    for rows in rows_list:
        res, _ = _worker((tables, rows, dim, B, L, alpha, 0.02, samples, steps, warmup, 0, 7))
        bags = sum(b for b, _ in res)
        secs = sum(t for _, t in res)
        out[rows] = bags / secs
    return out
