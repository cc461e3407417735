"""Pooled-result cache keyspace on the GPU (cache.py:204-223,
ranker.py:238-249,401-414) vs the reference: the golden runs recorded with
pooled_results=True (tests/golden/pooled.json) are replayed through the GPU
Ranker; per-batch metrics, counters, LRU order over row AND pooled keys,
used bytes (including the bytes the reference leaks on in-place re-puts)
and the eviction log must match exactly."""

import json
import os

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_12794_b200 as P
    return P


def _dev_key(k):
    """Golden key -> the GPU cache's decoded key."""
    if k[0] == "pooled":
        return ("pooled", O.pooled_fingerprint(k[1], k[2], k[3])[0])
    return tuple(k)


def _build(P, rec):
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    metas = [P.TableMeta(*m) for m in rec["metas"]]
    placement = [P.ShardSpec(*s) for s in rec["placement"]]
    dep = P.init_store(metas, placement, 0)
    rt = P.build_routing(metas, placement)
    cc = rec["cache"]
    cache = C.AdaptiveCache(cc["budget"], admission=cc["admission"], pooled_results=True, record_evictions=True,
                            max_dim=16)
    policy = C.CachePolicy(C.MemoryModel(*cc["model"]), cc["hyst"])
    w, hi, lo = cc["tracker"]
    tracker = C.LoadTracker(window=w, high_watermark=hi, low_watermark=lo)
    rk = Ranker(dep, rt, None, RankerParams(pushdown_threshold=rec["threshold"], admit_per_batch=cc["admit"]),
                cache=cache, policy=policy, tracker=tracker)
    return dep, rk


@pytest.mark.parametrize("parallel", [True, False])
@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_pooled_ranker_replays_reference(P, golden_dir, which, parallel):
    rec = json.load(open(os.path.join(golden_dir, "pooled.json")))["ranker"][which]
    dep, rk = _build(P, rec)
    rk.cache.set_parallel_offers(parallel)
    for bi, lookups in enumerate(rec["batches"]):
        batch = P.Batch(bi, bi, [P.LookupRequest([P.Feature(t, P.PoolingOp(op), ix) for t, op, ix in lk])
                                 for lk in lookups])
        res = rk.execute_batch(batch)
        m = rk.batch_metrics[-1]
        ref = rec["metrics"][bi]
        assert (m.cache_hits, m.cache_misses, m.pushdown_groups, m.pushdown_rows, m.raw_rows) == \
            (ref["hits"], ref["misses"], ref["pushdown_groups"], ref["pushdown_rows"], ref["raw_rows"]), bi
        assert m.subrequests == ref["subrequests"]
        assert (m.cache_budget, m.cache_used) == (ref["budget"], ref["used"]), bi
        for li, (lk, r) in enumerate(zip(lookups, res)):
            assert [r.cache_hits, r.pushdown_groups, r.pushdown_rows, r.raw_rows] == rec["counters"][bi][li]
            for fp, (t, op, ix) in enumerate(lk):
                ref_vec = np.array(rec["results"][bi][li][fp], dtype=np.uint32).view(np.float32)
                assert O.within_tolerance(ref_vec, r.vectors[fp])
                flat = O.pool_flat(O.rows_of(0, t, dep.meta(t).dim, ix), op)
                assert flat.tobytes() == r.vectors[fp].tobytes()
        assert rk.cache.lru_keys() == [_dev_key(k) for k in rec["per_batch_lru"][bi]], bi
        assert rk.cache.used_bytes == rec["per_batch_used"][bi]
    assert rk.cache.eviction_log == [_dev_key(k) for k in rec["evictions"]]
    print(rec["name"], "parallel put calls:", rk.cache._scalars()["n_par_puts"], "of", len(rec["batches"]))


def test_pooled_api_matches_reference(P, golden_dir):
    """cache.py:204-223 through the reference-facing API, incl. test_cache.py:222-228
    (keyed by the sorted multiset) and an in-place re-put."""
    from paper_2410_12794_b200.cache import AdaptiveCache
    api = json.load(open(os.path.join(golden_dir, "pooled.json")))["api"]
    c = AdaptiveCache(3 * 64, pooled_results=True, record_evictions=True, max_dim=16)
    v = lambda x: np.full(16, x, np.float32)
    S, M = P.PoolingOp.SUM, P.PoolingOp.MEAN
    c.pooled_put(0, S, [2, 1], v(9.0))
    c.offer(0, 5, v(1.0))
    c.pooled_put(0, S, [1, 2], v(7.0))
    got = c.pooled_get(0, S, [1, 2])
    c.pooled_put(1, M, [3], v(4.0))
    assert [list(k[:3]) + ([list(k[3])] if len(k) > 3 else []) for k in c.lru_keys()] == api["lru"]
    assert (c.used_bytes, c.tick) == (api["used"], api["tick"])
    assert [float(x) for x in got] == api["got"]
    assert [list(k) if k[0] != "pooled" else ["pooled", k[1], k[2], list(k[3])] for k in c.eviction_log] == \
        api["evictions"]
    # disabled by default (test_cache.py:214-219): no tick, None
    d = AdaptiveCache(10 * 64, max_dim=16)
    d.pooled_put(0, S, [1, 2], v(1.0))
    assert d.pooled_get(0, S, [1, 2]) is None and d.tick == 0


def test_pooled_result_cache_short_circuits(P):
    """test_ranker.py:272-283: the second identical request is served from the
    pooled keyspace without touching any shard."""
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker
    metas = [P.TableMeta(0, 100, 16)]
    placement = [P.ShardSpec(0, 0, 100, 0)]
    dep = P.init_store(metas, placement, 0)
    rk = Ranker(dep, P.build_routing(metas, placement), None, cache=C.AdaptiveCache(10 ** 6, pooled_results=True,
                                                                                   max_dim=16))
    b1 = P.Batch(0, 0, [P.LookupRequest([P.Feature(0, P.PoolingOp.SUM, [10, 11, 12, 13])])])
    b2 = P.Batch(1, 1, [P.LookupRequest([P.Feature(0, P.PoolingOp.SUM, [13, 12, 11, 10])])])
    r1 = rk.execute_batch(b1)
    r2 = rk.execute_batch(b2)
    assert np.array_equal(r1[0].vectors[0], r2[0].vectors[0])
    assert r2[0].cache_hits == 4 and r2[0].pushdown_groups == 0 and r2[0].raw_rows == 0
    assert rk.batch_metrics[-1].subrequests == 0


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_parallel_puts_equal_sequential(P, seed):
    """Closed-form parallel pooled_put (uniform size) == the ordered loop:
    random put streams with many re-puts, pre-filled caches and evictions."""
    from paper_2410_12794_b200.cache import AdaptiveCache
    rng = np.random.default_rng(seed)
    D = 16
    budget = 64 * int(rng.integers(50, 400))
    caches = [AdaptiveCache(budget, pooled_results=True, record_evictions=True, max_dim=D) for _ in range(2)]
    caches[1].set_parallel_offers(False)
    dev = torch.device("cuda")
    par_calls = []
    for step in range(12):
        n = int(rng.integers(1, 600))
        universe = int(rng.integers(5, 2000))
        ids = rng.integers(0, universe, n)
        if step % 4 != 3:  # keys resident at call start force the ordered loop; mostly avoid them
            ids = ids + (step + 1) * 1_000_000
        ka = torch.from_numpy((ids.astype(np.uint64) * np.uint64(2654435761) | np.uint64(1 << 63)).view(np.int64))
        kb = torch.from_numpy(ids.astype(np.int64) * 7 + 1)
        rows = torch.from_numpy(rng.standard_normal((n, D)).astype(np.float32)).to(dev)
        row_key = int(rng.integers(0, 50))
        for c in caches:
            c.pooled_put_many(ka.to(dev), kb.to(dev), rows, D * 4)
            if step % 3 == 1:  # a row offer in between (mixed keyspaces)
                c.offer(0, row_key, np.ones(D, np.float32))
        s0, s1 = caches[0]._scalars(), caches[1]._scalars()
        for k in ("used", "tick", "entries", "err"):
            assert s0[k] == s1[k], (step, k)
        assert caches[0].lru_entries() == caches[1].lru_entries(), step
        assert caches[0].eviction_log == caches[1].eviction_log
        par_calls.append(s0["n_par_puts"])
        keys = [k for k, _, _ in caches[0].lru_entries() if k[0] == "pooled"]
        if keys:
            ka_l = torch.tensor([k[1] - (1 << 64) for k in keys], dtype=torch.int64, device=dev)
            outs = []
            for c in caches:
                out = torch.zeros((len(keys), D), dtype=torch.float32, device=dev)
                slot = torch.empty(len(keys), dtype=torch.int32, device=dev)
                c._L.fx_cache_lookup(c._h, ka_l.data_ptr(), len(keys), out.data_ptr(), D, slot.data_ptr(), None)
                assert bool((slot >= 0).all())
                outs.append(out.cpu())
            assert torch.equal(outs[0], outs[1])
    assert caches[1]._scalars()["n_par_puts"] == 0
    assert par_calls[-1] > 0  # the closed form resolved at least some calls
