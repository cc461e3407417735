"""Pin the vectorised canonical-order cache (oracle/cache_vec.py) against the
per-occurrence restatement (oracle.restate.CacheOracle / PipelineOracle),
which tests/test_oracle_golden.py pins to the reference's own sessions."""

import numpy as np
import pytest

import oracle as O
from oracle.cache_vec import RowCacheVec, RowPipelineVec, keys_sample_major
from paper_2410_12794_b200.workload import DlrmBatchGen


def _run_both(rows, dim, B, pool, alpha, budget_rows, threshold, admission, n_batches, seed, policy_caps=None):
    T = len(rows)
    S = dim * 4
    gen = DlrmBatchGen(rows, alpha, B, pool, seed=seed)
    placement = O.Placement.from_specs({t: n for t, n in enumerate(rows)}, [(t, 0, n, 0) for t, n in enumerate(rows)])
    caps = policy_caps or [budget_rows * S] * n_batches
    model_o = O.MemoryModelO(caps[0] + 1000 + B, 1000, 1)
    model_v = O.MemoryModelO(caps[0] + 1000 + B, 1000, 1)
    co = O.CacheOracle(budget_rows * S, admission)
    po = O.PipelineOracle(0, {t: dim for t in range(T)}, placement, threshold=threshold, cache=co,
                          policy=O.CachePolicyO(model_o), tracker=O.LoadTrackerO(16, 10 ** 9, 0))
    cv = RowCacheVec(budget_rows * S, S, admission, record_evictions=True)
    pv = RowPipelineVec(cv, threshold, policy=O.CachePolicyO(model_v), tracker=O.LoadTrackerO(16, 10 ** 9, 0))
    for i in range(n_batches):
        model_o.cap = model_v.cap = caps[i] + 1000 + B   # budget moves: resize shrink / grow + stage
        hb = gen.next()
        lookups = hb.to_lists()
        bb = O.bag_batch_from_lists(lookups, batch_id=i)
        po.run(bb)
        keys, lens = keys_sample_major(hb.indices, hb.offsets, hb.feature_tables, B)
        pv.run(keys, lens, B, batch_id=i)
        mo, mv = po.metrics[-1], pv.metrics[-1]
        for k in ("hits", "misses", "pushdown_groups", "pushdown_rows", "raw_rows"):
            assert mo[k] == mv[k], (i, k, mo[k], mv[k])
        lru_o = [(t << 40) | r for (t, r) in co.entries]
        assert lru_o == cv.keys.tolist(), i
        assert [e[0] for e in co.entries.values()] == cv.ticks.tolist(), i
        assert [e[2] for e in co.entries.values()] == cv.hits_e.tolist(), i
        assert co.tick == cv.tick and co.used == cv.used and co.budget == cv.budget
        sk_o = sorted(((t << 40) | r, v) for (t, r), v in co.sketch.items())
        assert [k for k, _ in sk_o] == cv.sk_keys.tolist(), i
        assert [v for _, v in sk_o] == cv.sk_vals.tolist(), i
        assert [(t << 40) | r for (t, r) in co.evictions] == cv.evictions, i
        assert [(t << 40) | r for (t, r), _ in co.pending] == cv.pending, i
    return cv


@pytest.mark.parametrize("threshold", [None, 2])
@pytest.mark.parametrize("admission", ["sketch", "always"])
def test_vec_cache_matches_restatement(threshold, admission):
    cv = _run_both((2000, 3000, 500), 16, 48, (1, 6), 1.0, 120, threshold, admission, 10, seed=3)
    assert len(cv) > 0


def test_vec_cache_resize_shrink_grow_stage():
    caps = [16 * 4 * b for b in (200, 200, 90, 90, 300, 300, 300, 40, 400, 400)]
    _run_both((1500, 800), 16, 40, (1, 8), 0.9, 200, None, "sketch", 10, seed=11, policy_caps=caps)


def test_vec_cache_tiny_budget_evicts_own_accepts():
    # budget smaller than one batch's candidates: accepts evict accepts of the
    # same offer call (V = entries ++ accepted candidates)
    _run_both((5000,), 8, 64, (3, 3), 0.6, 7, None, "sketch", 6, seed=5)
    _run_both((5000,), 8, 64, (3, 3), 0.6, 7, None, "always", 6, seed=5)


def test_vec_cache_trickle_staging_fills():
    # threshold 2 pushes most misses down: the cache fills through the
    # 64-row stage_hot_admissions trickle and apply_pending (ranker.py:439-441)
    cv = _run_both((1500, 800), 16, 40, (1, 8), 0.9, 300, 2, "sketch", 10, seed=11)
    assert len(cv) == 300


def _golden_pipeline(golden_dir):
    import json
    import os
    return json.load(open(os.path.join(golden_dir, "pipeline.json")))


def _batch_keys(lookups):
    keys, lens = [], []
    for feats in lookups:
        for t, _op, ix in feats:
            keys.extend((int(t) << 40) | int(i) for i in ix)
            lens.append(len(ix))
    return np.array(keys, np.uint64), np.array(lens, np.int64)


def test_vec_pipeline_depth_matches_reference(golden_dir):
    """pipeline_depth 2/3 (ranker.py:161-182) replayed by the vectorised
    oracle's start/finish split reproduces the reference Ranker's metrics,
    final LRU order + ticks, eviction log and sketch (tests/golden/pipeline.json)."""
    for rec in _golden_pipeline(golden_dir):
        c = rec["cache"]
        S = rec["metas"][0][2] * 4
        cv = RowCacheVec(c["budget"], S, c["admission"], record_evictions=True)
        pv = RowPipelineVec(cv, rec["threshold"], policy=O.CachePolicyO(O.MemoryModelO(*c["model"]), c["hyst"]),
                            tracker=O.LoadTrackerO(*c["tracker"]), admit_per_batch=c["admit"])
        batches = [(*_batch_keys(lk), len(lk), i) for i, lk in enumerate(rec["batches"])]
        pv.run_trace(batches, depth=rec["depth"])
        for got, ref in zip(pv.metrics, rec["metrics"]):
            for k in ("batch_id", "hits", "misses", "pushdown_groups", "pushdown_rows", "raw_rows", "subrequests",
                      "load_level", "budget", "used"):
                assert got[k] == ref[k], (rec["name"], k, got[k], ref[k])
        assert cv.keys.tolist() == [(t << 40) | r for t, r in rec["lru"]], rec["name"]
        assert cv.ticks.tolist() == rec["ticks"], rec["name"]
        assert cv.evictions == [(t << 40) | r for t, r in rec["evictions"]], rec["name"]
        assert cv.sk_keys.tolist() == [(t << 40) | r for t, r, _ in rec["final_sketch"]], rec["name"]
        assert cv.sk_vals.tolist() == [v for _, _, v in rec["final_sketch"]], rec["name"]
