"""Ranker mirror (GPU pipeline) vs the reference Ranker, replaying the
golden runs recorded from the reference (tests/golden/ranker.json): per
batch metrics, per-lookup counters, cache LRU order after every batch,
eviction log and final sketch must match exactly; pooled vectors must be
within the reference tolerance of the reference's own results and
bit-identical to the flat f64 oracle."""

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


def _build(P, rec, fused=True):
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    metas = [P.TableMeta(*m) for m in rec["metas"]]
    placement = [P.ShardSpec(*s) for s in rec["placement"]]
    dep = P.init_store(metas, placement, 0)
    rt = P.build_routing(metas, placement)
    cache = policy = tracker = None
    admit = 64
    if "cache" in rec:
        cc = rec["cache"]
        cache = C.AdaptiveCache(cc["budget"], admission=cc["admission"], record_evictions=True, max_dim=16)
        policy = C.CachePolicy(C.MemoryModel(*cc["model"]), cc["hyst"])
        w, hi, lo = cc["tracker"]
        tracker = C.LoadTracker(window=w, high_watermark=hi, low_watermark=lo)
        admit = cc["admit"]
    rk = Ranker(dep, rt, None, RankerParams(pushdown_threshold=rec["threshold"], admit_per_batch=admit),
                cache=cache, policy=policy, tracker=tracker, fused=fused)
    return dep, rk


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_ranker_replays_reference(P, golden_dir, which, fused):
    """fused=True: the sync-free fused batch step (csrc/fx_step.cu) wherever
    the deployment is in its domain (the 1-server cache runs); False: the
    staged pipeline."""
    recs = json.load(open(os.path.join(golden_dir, "ranker.json")))
    rec = recs[which]
    dep, rk = _build(P, rec, fused)
    # these runs mix row sizes (dims 16 and 8): the staged pipeline serves them
    # either way; tests/golden/pipeline.json replays the fused step
    for bi, lookups in enumerate(rec["batches"]):
        batch = P.Batch(bi, bi, [P.LookupRequest([P.Feature(t, P.PoolingOp(op), ix) for t, op, ix in lk])
                                 for lk in lookups])
        res = rk.execute_batch(batch)
        m = rk.batch_metrics[-1]
        ref = rec["metrics"][bi]
        assert (m.cache_hits, m.cache_misses, m.pushdown_groups, m.pushdown_rows, m.raw_rows) == \
            (ref["hits"], ref["misses"], ref["pushdown_groups"], ref["pushdown_rows"], ref["raw_rows"]), bi
        assert m.subrequests == ref["subrequests"]
        assert m.load_level == ref["load_level"]
        assert (m.cache_budget, m.cache_used) == (ref["budget"], ref["used"])
        for li, (lk, r) in enumerate(zip(lookups, res)):
            assert [r.cache_hits, r.pushdown_groups, r.pushdown_rows, r.raw_rows] == rec["counters"][bi][li]
            for fp, (t, op, ix) in enumerate(lk):
                ref_vec = np.array(rec["results"][bi][li][fp], dtype=np.uint32).view(np.float32)
                assert O.within_tolerance(ref_vec, r.vectors[fp])
                flat = O.pool_flat(O.rows_of(0, t, dep.meta(t).dim, ix), op)
                assert flat.tobytes() == r.vectors[fp].tobytes()
        if rk.cache is not None:
            assert [list(k) for k in rk.cache.lru_keys()] == rec["per_batch_lru"][bi], bi
    if rk.cache is not None:
        assert [list(k) for k in rk.cache.eviction_log] == rec["evictions"]
        assert sorted([[k[0], k[1], v] for k, v in rk.cache.sketch.ranked()]) == rec["final_sketch"]


def test_ranker_validation_error_message(P):
    from paper_2410_12794_b200.ranker import Ranker
    metas = [P.TableMeta(0, 200, 8)]
    placement = [P.ShardSpec(0, 0, 100, 0), P.ShardSpec(0, 100, 200, 1)]
    dep = P.init_store(metas, placement, 0)
    rk = Ranker(dep, P.build_routing(metas, placement))
    batch = P.Batch(0, 0, [P.LookupRequest([P.Feature(0, P.PoolingOp.SUM, [5, 9])]),
                           P.LookupRequest([P.Feature(0, P.PoolingOp.SUM, [5, 999])])])
    with pytest.raises(P.LookupValidationError, match="batch 0, lookup 1: index 999"):
        rk.execute_batch(batch)


def test_counters_examples(P):
    """2 cached + 3 on S0 (pushdown) + 1 on S1 (raw) -> counters (2, 1, 1) (test_ranker.py:89-101)."""
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker
    metas = [P.TableMeta(0, 200, 64)]
    placement = [P.ShardSpec(0, 0, 100, 0), P.ShardSpec(0, 100, 200, 1)]
    dep = P.init_store(metas, placement, 0)
    cache = C.AdaptiveCache(10**6, admission="always", max_dim=64)
    rk = Ranker(dep, P.build_routing(metas, placement), cache=cache)
    for i in (5, 150):
        cache.offer(0, i, dep.get_row(0, i))
    res = rk.execute_batch(P.Batch(0, 0, [P.LookupRequest([P.Feature(0, P.PoolingOp.MEAN, [5, 150, 10, 11, 12, 120])])]))
    assert res[0].counters == (2, 1, 1) and res[0].pushdown_rows == 3
    ref = O.pool_flat(O.rows_of(0, 0, 64, [5, 150, 10, 11, 12, 120]), "mean")
    assert O.within_tolerance(ref, res[0].vectors[0])


def test_execute_csr_and_fused_path_match_execute_batch(P):
    """The batched CSR front end (execute_csr) and the single-fused-launch
    pooling (hits_from_cache=False) reproduce execute_batch exactly: pooled
    vectors bit-for-bit, counters, metrics and cache state."""
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen
    rows, D, B = (3000, 500, 1200), 32, 48
    metas = [P.TableMeta(t, n, D) for t, n in enumerate(rows)]
    placement = [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(rows)]
    dep = P.init_store(metas, placement, 0)
    ops = ("sum", "mean", "sum")

    def mk(hfc):
        cache = C.AdaptiveCache(150 * D * 4, admission="sketch", max_dim=D, record_evictions=True)
        model = C.MemoryModel(150 * D * 4 + 1000, 1000, 1)
        return Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=None,
                                                                                 admit_per_batch=8),
                      cache=cache, policy=C.CachePolicy(model), tracker=C.LoadTracker(4, 512, 16),
                      hits_from_cache=hfc)
    ra, rb, rc = mk(True), mk(True), mk(False)
    gen = DlrmBatchGen(rows, 1.1, B, (1, 9), seed=4, ops=ops)
    for bi in range(5):
        hb = gen.next()
        lk = hb.to_lists()
        batch = P.Batch(bi, bi, [P.LookupRequest([P.Feature(t, P.PoolingOp(op), ix) for t, op, ix in l]) for l in lk])
        res = ra.execute_batch(batch)
        idx, offs = torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda()
        pb, cb = rb.execute_csr(idx, offs, hb.feature_tables, hb.feature_ops, B, batch_id=bi)
        pc, cc = rc.execute_csr(idx, offs, hb.feature_tables, hb.feature_ops, B, batch_id=bi)
        ref = np.stack([np.concatenate(r.vectors) for r in res])
        assert np.array_equal(ref, pb.cpu().numpy()) and np.array_equal(ref, pc.cpu().numpy())
        ma, mb, mc = ra.batch_metrics[-1], rb.batch_metrics[-1], rc.batch_metrics[-1]
        for m in (mb, mc):
            assert (m.cache_hits, m.cache_misses, m.raw_rows, m.subrequests) == \
                (ma.cache_hits, ma.cache_misses, ma.raw_rows, ma.subrequests)
        # device-event latency / start time on every path (BatchMetrics, ranker.py:60-72)
        assert all(m.latency > 0 and m.started_at >= 0 for m in (ma, mb, mc))
        hits_sm = np.array([r.cache_hits for r in res])
        assert np.array_equal(cb["cache_hits"].view(len(rows), B).sum(0).cpu().numpy(), hits_sm)
        assert ra.cache.lru_entries() == rb.cache.lru_entries() == rc.cache.lru_entries()
    assert ra.batch_metrics[-1].cache_hits > 0
