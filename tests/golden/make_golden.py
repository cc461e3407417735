"""Generate golden fixtures by running the REFERENCE embserve package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference read-only from /root/reference/pkg/src and writes
small .npz/.json fixtures next to this file. Nothing at test/bench time
reads /root/reference: the fixtures are committed and travel with the repo.
"""

import json
import os
import sys
from collections import OrderedDict

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from embserve.cache import AdaptiveCache, CachePolicy, LoadTracker, MemoryModel  # noqa: E402
from embserve.pooling import PartialResult, PoolingOp, combine_partials, pool_flat  # noqa: E402
from embserve.ranker import Ranker, RankerParams  # noqa: E402
from embserve.requests import Batch, Feature, LookupRequest  # noqa: E402
from embserve.routing import build_routing, group_by_server  # noqa: E402
from embserve.store import ShardSpec, TableMeta, init_store, row_values, table_block  # noqa: E402
from embserve.transport.topology import assign_mapping_aware, create_connections  # noqa: E402
from embserve.transport.virtual import EventLoop, TransportParams, VirtualTransport  # noqa: E402
from embserve.workload import (CoOccurrence, Fluctuation, TableWorkload, WorkloadConfig,  # noqa: E402
                               ZipfSampler, generate_trace, save_trace)


def prf_fixtures():
    cases = [(0, 0, 64, 0, 16), (7, 3, 16, 1000, 1008), (12345, 5, 128, 9_999_996, 10_000_000),
             (2**31, 99, 1, 0, 32), (0, 0, 3, 5, 9), (11, 0, 3, 0, 6), (0, 25, 128, 5_461_300, 5_461_306),
             (2**63 + 5, 1, 256, 3, 5)]
    out = {}
    for i, (seed, t, d, s, e) in enumerate(cases):
        out[f"case{i}"] = np.array([seed % 2**64, t, d, s, e], dtype=np.uint64)
        out[f"block{i}"] = table_block(seed, t, d, s, e)
    # spot rows via row_values (store.py:77-79)
    out["rowv"] = np.stack([row_values(3, 2, r, 64) for r in (0, 1, 77, 99_999)])
    np.savez_compressed(os.path.join(HERE, "prf.npz"), **out)


def pool_fixtures():
    rng = np.random.default_rng(1234)
    out = {}
    # partial_pool bit-exact (store.py:184-193 / test_store.py:132-149)
    k = 0
    for dim in (1, 2, 3, 5, 9, 16, 64, 128, 256):
        rows = int(rng.integers(1, 50))
        seed = int(rng.integers(0, 2**31))
        dep = init_store([TableMeta(0, rows, dim)], [ShardSpec(0, 0, rows, 0)], seed=seed)
        for _ in range(4):
            n = int(rng.integers(1, 41))
            idx = rng.integers(0, rows, size=n).astype(np.int64)
            pr = dep.servers[0].partial_pool(0, [int(i) for i in idx], PoolingOp.SUM)
            out[f"pp{k}_meta"] = np.array([seed, rows, dim], np.int64)
            out[f"pp{k}_idx"] = idx
            out[f"pp{k}_vec"] = pr.vector
            out[f"pp{k}_raw"] = dep.servers[0].lookup_rows(0, [int(i) for i in idx])
            k += 1
    out["n_pp"] = np.array([k])
    # pool_flat / combine_partials on random rows + partitions (test_acceptance.py:45-77 style)
    k = 0
    for _ in range(160):
        dim = int(rng.integers(1, 70))
        n = int(rng.integers(1, 33))
        rows = (rng.random((n, dim)) * 2.0 - 1.0).astype(np.float32)
        if rng.random() < 0.1:
            rows *= np.float32(1e6) * rng.random((n, 1)).astype(np.float32)
        op = PoolingOp.SUM if rng.random() < 0.5 else PoolingOp.MEAN
        owners = rng.integers(0, int(rng.integers(1, 7)), size=n)
        partials, raw_pos, parts = [], [], []
        for g in np.unique(owners):
            mem = np.nonzero(owners == g)[0]
            if rng.random() < 0.6:
                acc = np.zeros(dim, np.float64)
                for i in mem:
                    acc += rows[i]
                partials.append(PartialResult(vector=acc.astype(np.float32), count=int(mem.size), source=int(g)))
                parts.append(int(g))
            else:
                raw_pos.extend(int(i) for i in mem)
        raw = [rows[i] for i in sorted(raw_pos)]
        out[f"c{k}_rows"] = rows
        out[f"c{k}_owner"] = owners
        out[f"c{k}_pushed"] = np.array(parts, np.int64)
        out[f"c{k}_op"] = np.array([0 if op is PoolingOp.SUM else 1])
        out[f"c{k}_comb"] = combine_partials(partials, raw, op)
        out[f"c{k}_flat"] = pool_flat(list(rows), op)
        k += 1
    out["n_c"] = np.array([k])
    # cancellation / ordering example (test_pooling.py:95-101)
    a = PartialResult(vector=np.array([1e8], np.float32), count=1, source=2)
    b = PartialResult(vector=np.array([-1e8], np.float32), count=1, source=0)
    c = PartialResult(vector=np.array([1.5], np.float32), count=1, source=1)
    out["order_example"] = combine_partials([c, a, b], [], PoolingOp.SUM)
    np.savez_compressed(os.path.join(HERE, "pool.npz"), **out)


def routing_fixtures():
    rng = np.random.default_rng(7)
    cases = []
    for trial in range(12):
        num_rows = int(rng.integers(50, 5000))
        n_cuts = int(rng.integers(0, min(7, num_rows - 1) + 1))
        cuts = sorted(rng.choice(np.arange(1, num_rows), size=n_cuts, replace=False).tolist()) if n_cuts else []
        bounds = [0] + [int(c) for c in cuts] + [num_rows]
        placement = [ShardSpec(0, bounds[i], bounds[i + 1], int(rng.integers(0, 16)))
                     for i in range(len(bounds) - 1)]
        rt = build_routing([TableMeta(0, num_rows, 4)], placement)
        idx = rng.integers(0, num_rows, size=500)
        res = rt.resolve_many(0, idx)
        feat = [int(i) for i in rng.integers(0, num_rows, size=int(rng.integers(1, 30)))]
        groups = group_by_server(rt, LookupRequest(features=[Feature(0, PoolingOp.SUM, feat)]))
        cases.append(dict(
            num_rows=num_rows,
            placement=[[s.table_id, s.start, s.end, s.server_id] for s in placement],
            entries=rt.entries(0),
            idx=[int(i) for i in idx], servers=[int(s) for s in res],
            feature=feat,
            groups=[[g.server_id, g.items[0].indices, g.items[0].positions] for g in groups],
        ))
    with open(os.path.join(HERE, "routing.json"), "w") as fh:
        json.dump(cases, fh)


def zipf_fixtures():
    out = {}
    for i, (n, a, seed, k) in enumerate([(100_000, 1.05, 0, 4096), (1000, 0.0, 3, 2000), (10, 1.2, 9, 500),
                                          (33_762, 0.6, 1, 3000)]):
        out[f"meta{i}"] = np.array([n, a, seed, k], np.float64)
        out[f"s{i}"] = ZipfSampler(n, a).sample(np.random.default_rng(seed), k)
    np.savez_compressed(os.path.join(HERE, "zipf.npz"), **out)


def cache_fixtures():
    """Scripted AdaptiveCache sessions (cache.py:164-352)."""
    rng = np.random.default_rng(99)
    sessions = []
    for sidx, adm in enumerate(("sketch", "always", "sketch")):
        RB = 16
        cache = AdaptiveCache(budget_bytes=40 * RB, admission=adm, record_evictions=True)
        fetch = lambda t, i: np.ones(4, np.float32)
        log = []
        sampler = ZipfSampler(300, 1.0)
        for step in range(25):
            cache.apply_pending_admissions()
            keys = [(int(rng.integers(0, 2)), int(r)) for r in sampler.sample(rng, 60)]
            hits = [cache.get(t, r) is not None for t, r in keys]
            seen = OrderedDict()
            for (t, r), h in zip(keys, hits):
                if not h:
                    seen.setdefault((t, r), None)
            offered = [bool(cache.offer(t, r, np.ones(4, np.float32))) for (t, r) in seen]
            op = None
            if step % 7 == 3:
                nb = int(cache.budget_bytes * (0.8 if sidx != 2 else 0.5))
                op = ["resize", nb]
                cache.resize(nb, fetcher=fetch, row_bytes_of=lambda t: RB)
            elif step % 7 == 5:
                nb = int(cache.budget_bytes * 1.4)
                op = ["resize", nb]
                cache.resize(nb, fetcher=fetch, row_bytes_of=lambda t: RB)
            staged = cache.stage_hot_admissions(fetch, lambda t: RB, limit=8)
            cache.sketch.age()
            log.append(dict(keys=keys, hits=hits, offers=list(map(list, seen)), offered=offered, op=op,
                            staged=[list(k) for k in staged],
                            lru=[list(k) for k in cache._entries],
                            ticks=[e.last_tick for e in cache._entries.values()],
                            budget=cache.budget_bytes, used=cache.used_bytes, tick=cache.tick,
                            sketch=sorted([[k[0], k[1], v] for k, v in cache.sketch._counts.items()])))
        sessions.append(dict(admission=adm, row_bytes=RB, budget0=40 * RB, steps=log,
                             evictions=[list(k) for k in cache.eviction_log]))
    with open(os.path.join(HERE, "cache.json"), "w") as fh:
        json.dump(sessions, fh)


def _ranker(metas, placement, cache=None, policy=None, tracker=None, threshold=2, conns=1, engines=1, units=1,
            admit=64):
    dep = init_store(metas, placement, 0)
    rt = build_routing(metas, placement)
    topo = create_connections(units, peers=dep.server_ids, conns_per_peer=conns)
    tr = VirtualTransport(EventLoop(), topo, assign_mapping_aware(topo, engines), TransportParams())
    return Ranker(dep, rt, tr, RankerParams(pushdown_threshold=threshold, admit_per_batch=admit),
                  cache=cache, policy=policy, tracker=tracker)


def ranker_fixtures():
    out = []
    rng = np.random.default_rng(5)
    # (a) 1 server, cache on (sketch), policy+tracker, threshold None and 2
    for thr in (None, 2):
        metas = [TableMeta(0, 2000, 16), TableMeta(1, 1500, 8)]
        placement = [ShardSpec(0, 0, 2000, 0), ShardSpec(1, 0, 1500, 0)]
        model = MemoryModel(gpu_capacity_bytes=64 * 300 + 1000, nn_fixed_bytes=1000, nn_per_sample_bytes=1)
        cache = AdaptiveCache(budget_bytes=64 * 300 - 64, admission="sketch", record_evictions=True)
        policy = CachePolicy(model=model, hysteresis_fraction=0.05)
        tracker = LoadTracker(window=4, high_watermark=512, low_watermark=16)
        rk = _ranker(metas, placement, cache, policy, tracker, threshold=thr, admit=16)
        batches = _zipf_batches(rng, metas, n_batches=8, lookups=(40, 70), L=(1, 8), alpha=1.0)
        out.append(_run_and_record(rk, batches, f"one_server_cache_thr{thr}", metas, placement))
    # (b) 3 servers, row-wise + table-wise mix, no cache, threshold 2
    metas = [TableMeta(0, 300, 8), TableMeta(1, 100, 5)]
    placement = [ShardSpec(0, 0, 120, 0), ShardSpec(0, 120, 200, 2), ShardSpec(0, 200, 300, 1),
                 ShardSpec(1, 0, 100, 1)]
    rk = _ranker(metas, placement, threshold=2, conns=2, engines=2, units=2)
    batches = _zipf_batches(rng, metas, n_batches=3, lookups=(20, 30), L=(1, 12), alpha=0.8, mean_p=0.5)
    out.append(_run_and_record(rk, batches, "three_server_nocache", metas, placement))
    with open(os.path.join(HERE, "ranker.json"), "w") as fh:
        json.dump(out, fh)


def pipeline_fixtures():
    """Ranker.run_trace with pipeline_depth 2 and 3 (ranker.py:161-182): up
    to `depth` batches in flight, so batch k+depth starts (apply_pending +
    probes) only after batch k finished (offers + maintenance). One server,
    one connection, one engine: batches finish in arrival order."""
    out = []
    rng = np.random.default_rng(21)
    for depth, thr in ((2, None), (3, None), (2, 2), (1, None), (1, 2)):
        metas = [TableMeta(0, 1500, 16), TableMeta(1, 900, 16)]
        placement = [ShardSpec(0, 0, 1500, 0), ShardSpec(1, 0, 900, 0)]
        budget = 64 * 150
        model = MemoryModel(gpu_capacity_bytes=budget + 1000 + 100, nn_fixed_bytes=1000, nn_per_sample_bytes=1)
        cache = AdaptiveCache(budget_bytes=budget, admission="sketch", record_evictions=True)
        policy = CachePolicy(model=model, hysteresis_fraction=0.05)
        tracker = LoadTracker(window=4, high_watermark=512, low_watermark=16)
        dep = init_store(metas, placement, 0)
        rt = build_routing(metas, placement)
        topo = create_connections(1, peers=dep.server_ids, conns_per_peer=1)
        tr = VirtualTransport(EventLoop(), topo, assign_mapping_aware(topo, 1), TransportParams())
        rk = Ranker(dep, rt, tr, RankerParams(pushdown_threshold=thr, admit_per_batch=8, pipeline_depth=depth),
                    cache=cache, policy=policy, tracker=tracker)
        batches = _zipf_batches(rng, metas, n_batches=7, lookups=(30, 50), L=(1, 6), alpha=1.0)
        rk.run_trace(batches)
        out.append(dict(
            name=f"pipeline_depth{depth}_thr{thr}", depth=depth, threshold=thr,
            metas=[[m.table_id, m.num_rows, m.dim] for m in metas],
            placement=[[s.table_id, s.start, s.end, s.server_id] for s in placement],
            cache=dict(budget=budget, admission="sketch",
                       model=[model.gpu_capacity_bytes, model.nn_fixed_bytes, model.nn_per_sample_bytes],
                       hyst=0.05, tracker=[4, 512, 16], admit=8),
            batches=[[[[f.table_id, f.op.value, f.indices] for f in lk.features] for lk in b.lookups]
                     for b in batches],
            metrics=[dict(batch_id=m.batch_id, hits=m.cache_hits, misses=m.cache_misses,
                          pushdown_groups=m.pushdown_groups, pushdown_rows=m.pushdown_rows, raw_rows=m.raw_rows,
                          load_level=m.load_level, budget=m.cache_budget, used=m.cache_used,
                          subrequests=m.subrequests) for m in rk.batch_metrics],
            results={str(b.batch_id): [[[float(x) for x in v.view(np.uint32).astype(np.float64)] for v in r.vectors]
                                       for r in rk.results[b.batch_id]] for b in batches},
            lru=[list(k) for k in cache._entries],
            ticks=[e.last_tick for e in cache._entries.values()],
            evictions=[list(k) for k in cache.eviction_log],
            final_sketch=sorted([[k[0], k[1], v] for k, v in cache.sketch._counts.items()])))
    with open(os.path.join(HERE, "pipeline.json"), "w") as fh:
        json.dump(out, fh)


def _key_json(k):
    if isinstance(k, tuple) and len(k) == 4 and k[0] == "pooled":
        return ["pooled", k[1], k[2], list(k[3])]
    return list(k)


def pooled_fixtures():
    """Ranker with the pooled-result keyspace on (cache.py:204-223,
    ranker.py:238-249,401-414), 1 server: small tables and short bags so
    bag multisets repeat within and across batches (pooled hits, in-place
    re-puts and their leaked bytes)."""
    out = []
    rng = np.random.default_rng(9)
    for thr, budget_rows, n_batches, name, rows0, L in ((2, 400, 6, "pooled_thr2", 40, (1, 3)),
                                                       (None, 300, 6, "pooled_thrNone", 40, (1, 3)),
                                                       (2, 40, 8, "pooled_churn", 40, (1, 3)),
                                                       (2, 60, 12, "pooled_leak", 6, (1, 1))):
        metas = [TableMeta(0, rows0, 16), TableMeta(1, 600, 16)]
        placement = [ShardSpec(0, 0, rows0, 0), ShardSpec(1, 0, 600, 0)]
        budget = 64 * budget_rows
        model = MemoryModel(gpu_capacity_bytes=budget + 1000 + 100, nn_fixed_bytes=1000, nn_per_sample_bytes=1)
        cache = AdaptiveCache(budget_bytes=budget, admission="sketch", pooled_results=True, record_evictions=True)
        policy = CachePolicy(model=model, hysteresis_fraction=0.05)
        tracker = LoadTracker(window=4, high_watermark=512, low_watermark=16)
        rk = _ranker(metas, placement, cache, policy, tracker, threshold=thr, admit=8)
        batches = _zipf_batches(rng, metas, n_batches=n_batches, lookups=(20, 30), L=L, alpha=1.2, mean_p=0.3)
        rec = dict(name=name, metas=[[m.table_id, m.num_rows, m.dim] for m in metas],
                   placement=[[s.table_id, s.start, s.end, s.server_id] for s in placement], threshold=thr,
                   cache=dict(budget=budget, admission="sketch",
                              model=[model.gpu_capacity_bytes, model.nn_fixed_bytes, model.nn_per_sample_bytes],
                              hyst=0.05, tracker=[4, 512, 16], admit=8),
                   batches=[], results=[], counters=[], metrics=[], per_batch_lru=[], per_batch_used=[],
                   raised_at=None)
        for b in batches:
            rec["batches"].append([[[f.table_id, f.op.value, f.indices] for f in lk.features] for lk in b.lookups])
            try:
                rk.execute_batch(b)
            except KeyError:
                rec["raised_at"] = b.batch_id
                break
            res = rk.results[b.batch_id]
            rec["results"].append([[[float(x) for x in v.view(np.uint32).astype(np.float64)] for v in r.vectors]
                                   for r in res])
            rec["counters"].append([[r.cache_hits, r.pushdown_groups, r.pushdown_rows, r.raw_rows] for r in res])
            m = rk.batch_metrics[-1]
            rec["metrics"].append(dict(hits=m.cache_hits, misses=m.cache_misses, pushdown_groups=m.pushdown_groups,
                                       pushdown_rows=m.pushdown_rows, raw_rows=m.raw_rows, load_level=m.load_level,
                                       budget=m.cache_budget, used=m.cache_used, subrequests=m.subrequests))
            rec["per_batch_lru"].append([_key_json(k) for k in rk.cache._entries])
            rec["per_batch_used"].append(rk.cache.used_bytes)
        rec["evictions"] = [_key_json(k) for k in rk.cache.eviction_log]
        out.append(rec)
    # API-level example (test_cache.py:222-228) plus an in-place re-put
    c = AdaptiveCache(budget_bytes=3 * 64, pooled_results=True, record_evictions=True)
    v = lambda x: np.full(16, x, np.float32)
    c.pooled_put(0, PoolingOp.SUM, [2, 1], v(9.0))
    c.offer(0, 5, v(1.0))
    c.pooled_put(0, PoolingOp.SUM, [1, 2], v(7.0))   # resident: replaced in place, used += 64
    got = c.pooled_get(0, PoolingOp.SUM, [1, 2])
    c.pooled_put(1, PoolingOp.MEAN, [3], v(4.0))       # evicts the LRU entry
    api = dict(lru=[_key_json(k) for k in c._entries], used=c.used_bytes, tick=c.tick,
               got=[float(x) for x in got], evictions=[_key_json(k) for k in c.eviction_log])
    with open(os.path.join(HERE, "pooled.json"), "w") as fh:
        json.dump(dict(ranker=out, api=api), fh)


def _zipf_batches(rng, metas, n_batches, lookups, L, alpha, mean_p=0.0):
    samplers = {m.table_id: ZipfSampler(m.num_rows, alpha) for m in metas}
    batches = []
    for b in range(n_batches):
        lk = []
        for _ in range(int(rng.integers(lookups[0], lookups[1] + 1))):
            feats = []
            for m in metas:
                n = int(rng.integers(L[0], L[1] + 1))
                op = PoolingOp.MEAN if rng.random() < mean_p else PoolingOp.SUM
                feats.append(Feature(m.table_id, op, [int(i) for i in samplers[m.table_id].sample(rng, n)]))
            lk.append(LookupRequest(features=feats))
        batches.append(Batch(batch_id=b, tick=b, lookups=lk))
    return batches


def _run_and_record(rk, batches, name, metas, placement):
    rec = dict(name=name, metas=[[m.table_id, m.num_rows, m.dim] for m in metas],
               placement=[[s.table_id, s.start, s.end, s.server_id] for s in placement],
               threshold=rk.params.pushdown_threshold, batches=[], results=[], metrics=[])
    if rk.cache is not None:
        rec["cache"] = dict(budget=rk.cache.budget_bytes, admission=rk.cache.admission,
                            model=[rk.policy.model.gpu_capacity_bytes, rk.policy.model.nn_fixed_bytes,
                                   rk.policy.model.nn_per_sample_bytes],
                            hyst=rk.policy.hysteresis_fraction,
                            tracker=[rk.tracker.window.maxlen, rk.tracker.high_watermark, rk.tracker.low_watermark],
                            admit=rk.params.admit_per_batch)
        rec["per_batch_lru"] = []
    for b in batches:
        rk.execute_batch(b)
        rec["batches"].append([[[f.table_id, f.op.value, f.indices] for f in lk.features] for lk in b.lookups])
        res = rk.results[b.batch_id]
        rec["results"].append([[[float(x) for x in v.view(np.uint32).astype(np.float64)] for v in r.vectors]
                               for r in res])
        rec.setdefault("counters", []).append([[r.cache_hits, r.pushdown_groups, r.pushdown_rows, r.raw_rows]
                                               for r in res])
        m = rk.batch_metrics[-1]
        rec["metrics"].append(dict(hits=m.cache_hits, misses=m.cache_misses, pushdown_groups=m.pushdown_groups,
                                   pushdown_rows=m.pushdown_rows, raw_rows=m.raw_rows, load_level=m.load_level,
                                   budget=m.cache_budget, used=m.cache_used, subrequests=m.subrequests))
        if rk.cache is not None:
            rec["per_batch_lru"].append([list(k) for k in rk.cache._entries])
    if rk.cache is not None:
        rec["evictions"] = [list(k) for k in rk.cache.eviction_log]
        rec["final_sketch"] = sorted([[k[0], k[1], v] for k, v in rk.cache.sketch._counts.items()])
    return rec


def trace_fixtures():
    """Reference generate_trace + save_trace output (workload.py:160-221)."""
    cfgs = {
        "trace_a.txt": (WorkloadConfig(tables=[TableWorkload(0, 1.0), TableWorkload(1, 0.5, weight=2.0, op=PoolingOp.MEAN)],
                                       lookups_per_batch=12, indices_per_lookup=(2, 9), features_per_lookup=2,
                                       fluctuation=Fluctuation(0.4, 5), duration_batches=6, seed=11,
                                       co_occurrence=CoOccurrence(3, 0.3)), {0: 500, 1: 60}),
        "trace_b.txt": (WorkloadConfig(tables=[TableWorkload(3, 1.2)], lookups_per_batch=7, indices_per_lookup=(4, 4),
                                       duration_batches=4, seed=2), {3: 1000}),
    }
    for name, (cfg, rows) in cfgs.items():
        save_trace(generate_trace(cfg, rows), os.path.join(HERE, name))


def report_fixtures():
    """bench/report.py: percentiles and the MetricsReport text/machine forms."""
    from embserve.bench.report import MetricsReport, RunMetrics, percentiles
    rng = np.random.default_rng(3)
    cases = [[], [5.0], [3.0, 1.0, 2.0], [float(x) for x in rng.random(37)], [float(x) for x in rng.integers(0, 9, 100)]]
    pct = [percentiles(c) for c in cases]
    rep = MetricsReport(experiment="golden-x", seed=7, backend="virtual", fingerprint="abc123",
                        config={"b": 2, "a": [1, 2]},
                        runs=[RunMetrics(label="r1", makespan=12.5, throughput=3.25, counters={"z": 1, "a": 2},
                                         latency_stages={"net": percentiles([1.0, 2.0, 4.0])},
                                         extras={"note": "x"}),
                              RunMetrics(label="r2")],
                        comparison={"speedup": 1.5}, invariants={"ok": True})
    with open(os.path.join(HERE, "report.json"), "w") as fh:
        json.dump(dict(cases=cases, percentiles=pct, machine=rep.to_machine(), text=rep.to_text()), fh)


if __name__ == "__main__":
    trace_fixtures()
    prf_fixtures()
    pool_fixtures()
    routing_fixtures()
    zipf_fixtures()
    cache_fixtures()
    ranker_fixtures()
    pooled_fixtures()
    report_fixtures()
    pipeline_fixtures()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
