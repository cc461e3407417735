"""The fused, sync-free cache batch step (csrc/fx_step.cu behind
Ranker.execute_csr / execute_batch / run_trace) against the oracles:

* cfg3-shaped batches (32 tables x 1M rows x dim 128, B=4096, L=20, Zipf
  alpha 0.6 and 1.2, cache 1% of rows, 6 batches) and batches that exercise
  the parallel decision chain with rejections, the pushdown threshold and
  "always" admission, against the vectorised canonical-order oracle
  (oracle/cache_vec.py, pinned to the reference by tests/test_cache_vec.py):
  per batch hits / misses / counters, the whole LRU (keys, ticks, hits), the
  eviction log, the sketch, the staged admissions, and sampled pooled
  vectors bit-identical to the flat f64 pool;
* pipeline_depth 2 and 3 (ranker.py:161-182) against the reference's own
  runs (tests/golden/pipeline.json);
* a rejected batch (bad index) raises the reference's message and leaves the
  cache untouched."""

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


@pytest.fixture(scope="module")
def dep_cfg3(P):
    T, N, D = 32, 1_000_000, 128
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    return P.init_store(metas, placement, 0)


def _assert_clean(rep):
    bad = [(r["batch"], r["bad"]) for r in rep if r["bad"]]
    assert not bad, bad


@pytest.mark.parametrize("alpha", [0.6, 1.2])
def test_cfg3_shaped_parity(P, dep_cfg3, alpha):
    from step_harness import run_compare
    rep, ctx = run_compare(tables=32, rows=1_000_000, dim=128, batch=4096, pooling=(20, 20), alpha=alpha,
                           cache_frac=0.01, n_batches=6, dep=dep_cfg3, check_vectors=512, log=lambda r: None)
    _assert_clean(rep)
    assert ctx["rk"]._fast and rep[-1]["hits"] > 0 and rep[-1]["accepted"] > 0


@pytest.mark.parametrize("alpha,frac", [(0.6, 0.05), (0.8, 0.02), (1.0, 0.05)])
def test_parallel_chain_with_rejections(P, dep_cfg3, alpha, frac):
    """B=1024: the candidates fit the eviction queue (parallel decisions) and
    the sketch rejects some of them (hard victims)."""
    from step_harness import run_compare
    rep, ctx = run_compare(tables=32, rows=1_000_000, dim=128, batch=1024, pooling=(20, 20), alpha=alpha,
                           cache_frac=frac, n_batches=6, dep=dep_cfg3, check_vectors=128, log=lambda r: None)
    _assert_clean(rep)
    sc = ctx["rk"]._step.scalars(0)
    assert sc["mode"] == 1  # MODE_PAR
    if alpha < 1.0:
        assert any(r["offers"] > r["accepted"] for r in rep)  # rejections happened


@pytest.mark.parametrize("threshold,admission", [(2, "sketch"), (None, "always"), (3, "always")])
def test_threshold_and_admission(P, dep_cfg3, threshold, admission):
    from step_harness import run_compare
    rep, _ = run_compare(tables=32, rows=1_000_000, dim=128, batch=512, pooling=(1, 12), alpha=1.0,
                         cache_frac=0.002, threshold=threshold, admission=admission, n_batches=5, dep=dep_cfg3,
                         check_vectors=64, log=lambda r: None)
    _assert_clean(rep)


def test_small_cache_sequential_path(P, dep_cfg3):
    """More accepts than entries (the eviction queue runs into this call's own
    accepts): the exact sequential path."""
    from step_harness import run_compare
    rep, ctx = run_compare(tables=32, rows=1_000_000, dim=128, batch=256, pooling=(5, 5), alpha=0.8,
                           cache_frac=0.00005, n_batches=4, dep=dep_cfg3, check_vectors=32, log=lambda r: None)
    _assert_clean(rep)
    assert ctx["rk"]._step.scalars(0)["mode"] == 2  # MODE_SEQ


@pytest.mark.parametrize("alpha,frac,depth", [(0.8, 0.01, 2), (1.0, 0.02, 3)])
def test_pipeline_depth_csr_stream(P, dep_cfg3, alpha, frac, depth):
    """execute_csr(sync=False) with pipeline_depth batches in flight vs the
    oracle's start/finish interleaving: candidates cached by a later batch's
    apply_pending take the dynamic-presence path."""
    from step_harness import run_compare
    rep, _ = run_compare(tables=32, rows=1_000_000, dim=128, batch=512, pooling=(1, 20), alpha=alpha,
                         cache_frac=frac, n_batches=7, dep=dep_cfg3, depth=depth, admit=512, log=lambda r: None)
    _assert_clean(rep)


@pytest.mark.parametrize("which", [0, 1, 2, 3, 4])
def test_pipeline_depth_replays_reference(P, golden_dir, which):
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    rec = json.load(open(os.path.join(golden_dir, "pipeline.json")))[which]
    metas = [P.TableMeta(*m) for m in rec["metas"]]
    placement = [P.ShardSpec(*s) for s in rec["placement"]]
    dep = P.init_store(metas, placement, 0)
    cc = rec["cache"]
    cache = C.AdaptiveCache(cc["budget"], admission=cc["admission"], record_evictions=True, max_dim=16)
    rk = Ranker(dep, P.build_routing(metas, placement), None,
                RankerParams(pushdown_threshold=rec["threshold"], admit_per_batch=cc["admit"],
                             pipeline_depth=rec["depth"]),
                cache=cache, policy=C.CachePolicy(C.MemoryModel(*cc["model"]), cc["hyst"]),
                tracker=C.LoadTracker(*cc["tracker"]))
    assert rk._fast
    batches = [P.Batch(bi, bi, [P.LookupRequest([P.Feature(t, P.PoolingOp(op), ix) for t, op, ix in lk])
                                for lk in lookups]) for bi, lookups in enumerate(rec["batches"])]
    rk.run_trace(batches)
    assert len(rk.batch_metrics) == len(rec["metrics"])
    for m, ref in zip(rk.batch_metrics, rec["metrics"]):
        assert (m.batch_id, m.cache_hits, m.cache_misses, m.pushdown_groups, m.pushdown_rows, m.raw_rows,
                m.subrequests, m.load_level, m.cache_budget, m.cache_used) == \
            (ref["batch_id"], ref["hits"], ref["misses"], ref["pushdown_groups"], ref["pushdown_rows"],
             ref["raw_rows"], ref["subrequests"], ref["load_level"], ref["budget"], ref["used"]), ref["batch_id"]
        assert m.latency > 0
    k, t, _ = cache.lru_arrays()
    assert k.tolist() == [(a << 40) | b for a, b in rec["lru"]]
    assert t.tolist() == rec["ticks"]
    assert [list(x) for x in cache.eviction_log] == rec["evictions"]
    assert sorted([[a[0], a[1], v] for a, v in cache.sketch.ranked()]) == rec["final_sketch"]
    for b in batches:
        for lk, r, refl in zip(b.lookups, rk.results[b.batch_id], rec["results"][str(b.batch_id)]):
            for f, got, refv in zip(lk.features, r.vectors, refl):
                ref_vec = np.array(refv, dtype=np.uint32).view(np.float32)
                assert O.within_tolerance(ref_vec, got)


def test_rejected_batch_leaves_cache_untouched(P):
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen
    T, N, D, B = 3, 20_000, 32, 64
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    dep = P.init_store(metas, placement, 0)
    budget = 500 * D * 4
    cache = C.AdaptiveCache(budget, max_dim=D, slot_capacity=501, sketch_capacity=50_000)
    rk = Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=None),
                cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1000 + B, 1000, 1)),
                tracker=C.LoadTracker(16, 10 ** 9, 0))
    gen = DlrmBatchGen((N,) * T, 1.0, B, (3, 8), seed=2)
    for i in range(3):
        hb = gen.next()
        rk.execute_csr(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(), hb.feature_tables,
                       hb.feature_ops, B, batch_id=i)
    before = (cache.lru_arrays(), cache.sketch.ranked_arrays(), cache._scalars(), list(rk.tracker.window))
    hb = gen.next()
    idx = hb.indices.copy()
    b_bad = 1 * B + 17                         # feature 1, sample 17
    idx[hb.offsets[b_bad] + 1] = N + 5
    with pytest.raises(P.LookupValidationError, match=f"batch 3, lookup 17: index {N + 5} out of range"):
        rk.execute_csr(torch.from_numpy(idx).cuda(), torch.from_numpy(hb.offsets).cuda(), hb.feature_tables,
                       hb.feature_ops, B, batch_id=3)
    after = (cache.lru_arrays(), cache.sketch.ranked_arrays(), cache._scalars(), list(rk.tracker.window))
    for x, y in zip(before[0] + before[1], after[0] + after[1]):
        assert np.array_equal(x, y)
    keep = ("budget", "used", "tick", "hits", "misses", "entries", "pending", "n_evlog", "sketch_live")
    assert {k: before[2][k] for k in keep} == {k: after[2][k] for k in keep} and before[3] == after[3]
    # the next good batch runs normally
    rk.execute_csr(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(), hb.feature_tables,
                   hb.feature_ops, B, batch_id=4)
    assert rk.batch_metrics[-1].batch_id == 4


def test_end_to_end_equivalence_check(P):
    """ranker.py:458-494 over a cfg1-shaped trace through the fused step."""
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams, end_to_end_equivalence_check
    from paper_2410_12794_b200.workload import DlrmBatchGen
    T, N, D, B = 8, 100_000, 64, 64
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    dep = P.init_store(metas, placement, 0)
    budget = 2000 * D * 4
    cache = C.AdaptiveCache(budget, max_dim=D, slot_capacity=2001, sketch_capacity=100_000)
    rk = Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=2),
                cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1000 + B, 1000, 1)),
                tracker=C.LoadTracker(16, 10 ** 9, 0))
    gen = DlrmBatchGen((N,) * T, 1.05, B, (20, 20), seed=1)
    batches = []
    for i in range(3):
        lk = gen.next().to_lists()
        batches.append(P.Batch(i, i, [P.LookupRequest([P.Feature(t, P.PoolingOp(op), ix) for t, op, ix in l])
                                      for l in lk]))
    rk.run_trace(batches)
    rep = end_to_end_equivalence_check(dep, batches, rk.results)
    assert rep.lookups_checked == 3 * B and rep.passed and rep.max_abs_diff == 0.0


@pytest.mark.parametrize("pooling", [(1, 9), (6, 6)])
def test_stream_host_matches_execute_csr(P, pooling):
    """The end-to-end host API returns the same pooled vectors and leaves the
    same cache state as device-resident execute_csr calls: fixed-size batches
    replay the two captured graphs, ragged ones mix graphs and eager batches."""
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen
    T, N, D, B = 4, 50_000, 32, 128
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    dep = P.init_store(metas, placement, 0)

    def mk():
        budget = 1500 * D * 4
        cache = C.AdaptiveCache(budget, max_dim=D, slot_capacity=1501, sketch_capacity=100_000)
        return Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=None),
                      cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1000 + B, 1000, 1)),
                      tracker=C.LoadTracker(16, 10 ** 9, 0))
    ra, rb = mk(), mk()
    gen = DlrmBatchGen((N,) * T, 1.0, B, pooling, seed=5)
    hbs = [gen.next() for _ in range(7)]
    ft, fo = hbs[0].feature_tables, hbs[0].feature_ops
    ref = [ra.execute_csr(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda(), ft, fo, B,
                          batch_id=i)[0].cpu().numpy() for i, h in enumerate(hbs)]
    pinned = [(torch.from_numpy(h.indices).pin_memory(), torch.from_numpy(h.offsets).pin_memory()) for h in hbs]
    got = [o.numpy().copy() for o in rb.stream_host(pinned, ft, fo, B)]
    assert len(got) == len(ref) and all(np.array_equal(a, b) for a, b in zip(ref, got))
    assert [m.cache_hits for m in ra.batch_metrics] == [m.cache_hits for m in rb.batch_metrics]
    for x, y in zip(ra.cache.lru_arrays(), rb.cache.lru_arrays()):
        assert np.array_equal(x, y)


def test_captured_batch_matches_eager(P):
    """Ranker.capture_csr: one CUDA graph per Ranker batch, replayed over
    static buffers, leaves exactly the state and metrics of eager batches."""
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen
    T, N, D, B = 4, 60_000, 64, 256
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    dep = P.init_store(metas, placement, 0)

    def mk():
        budget = 3000 * D * 4
        cache = C.AdaptiveCache(budget, max_dim=D, slot_capacity=3001, sketch_capacity=200_000,
                                record_evictions=True)
        return Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=None),
                      cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1000 + B, 1000, 1)),
                      tracker=C.LoadTracker(16, 10 ** 9, 0))
    ra, rb = mk(), mk()
    hbs = [b for b in (DlrmBatchGen((N,) * T, 0.9, B, (10, 10), seed=2).next() for _ in range(8))]
    ft, fo = hbs[0].feature_tables, hbs[0].feature_ops
    dev = [(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda()) for h in hbs]
    ref = [ra.execute_csr(*dev[i], ft, fo, B, batch_id=i)[0].cpu().numpy() for i in range(8)]
    rb.execute_csr(*dev[0], ft, fo, B, batch_id=0)
    sidx, soffs = dev[1][0].clone(), dev[1][1].clone()
    g = rb.capture_csr(sidx, soffs, ft, fo, B)
    got = [None]
    for i in range(1, 8):
        sidx.copy_(dev[i][0])
        soffs.copy_(dev[i][1])
        got.append(g.replay(batch_id=i).cpu().numpy())
    rb.sync()
    for i in range(1, 8):
        assert np.array_equal(ref[i], got[i]), i
    assert [m.cache_hits for m in ra.batch_metrics] == [m.cache_hits for m in rb.batch_metrics]
    for x, y in zip(ra.cache.lru_arrays(), rb.cache.lru_arrays()):
        assert np.array_equal(x, y)
    assert np.array_equal(ra.cache.eviction_log_array(), rb.cache.eviction_log_array())
