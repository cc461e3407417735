"""GPU Ranker (fused batch step) vs the vectorised canonical-order oracle
(oracle/cache_vec.py) on cfg3-shaped Zipf batches — shared by
tests/test_gpu_step.py and scripts/step_check.py (test infrastructure)."""

from __future__ import annotations

import time

import numpy as np
import torch

import oracle as O
from oracle.cache_vec import RowCacheVec, RowPipelineVec, keys_sample_major


def run_compare(tables=32, rows=1_000_000, dim=128, batch=1024, pooling=(20, 20), alpha=1.0, cache_frac=0.05,
                threshold=None, admission="sketch", n_batches=6, seed=7, admit=64, check_vectors=256,
                dep=None, fused=True, log=print, depth=1):
    import paper_2410_12794_b200 as P
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen

    T, N, D, B = tables, rows, dim, batch
    S = D * 4
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    if dep is None:
        dep = P.init_store(metas, placement, 0)
    gen = DlrmBatchGen((N,) * T, alpha, B, pooling, seed=seed)
    cache_rows = max(1, int(T * N * cache_frac))
    budget = cache_rows * S
    nnz_max = B * T * pooling[1]
    cache = C.AdaptiveCache(budget, admission=admission, max_dim=D, slot_capacity=cache_rows + 1,
                            sketch_capacity=6 * nnz_max, record_evictions=True)
    model = C.MemoryModel(budget + 1_000 + B, 1_000, 1)
    rk = Ranker(dep, P.build_routing(metas, placement), None,
                RankerParams(pushdown_threshold=threshold, admit_per_batch=admit, pipeline_depth=depth),
                cache=cache, policy=C.CachePolicy(model), tracker=C.LoadTracker(16, 10 ** 9, 0), fused=fused)
    cv = RowCacheVec(budget, S, admission, record_evictions=True)
    pv = RowPipelineVec(cv, threshold, policy=O.CachePolicyO(O.MemoryModelO(budget + 1_000 + B, 1_000, 1)),
                        tracker=O.LoadTrackerO(16, 10 ** 9, 0), admit_per_batch=admit)
    rng = np.random.default_rng(seed)
    report = []
    if depth > 1:
        # batches in flight: compare the whole run's metrics and final state
        # with the oracle's start/finish interleaving (ranker.py:161-182)
        hbs = [gen.next() for _ in range(n_batches)]
        rk.reserve(max(int(h.offsets[-1]) for h in hbs), max(h.offsets.size - 1 for h in hbs))
        for i, hb in enumerate(hbs):
            rk.execute_csr(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(),
                           hb.feature_tables, hb.feature_ops, B, batch_id=i, sync=False)
        rk.sync()
        pv.run_trace([(*keys_sample_major(hb.indices, hb.offsets, hb.feature_tables, B), B, i)
                      for i, hb in enumerate(hbs)], depth=depth)
        bad = []
        for mg, mo in zip(rk.batch_metrics, pv.metrics):
            if (mg.cache_hits, mg.cache_misses, mg.raw_rows) != (mo["hits"], mo["misses"], mo["raw_rows"]):
                bad.append(f"batch {mg.batch_id} metrics differ")
        k, t, h = cache.lru_arrays()
        if not (np.array_equal(k, cv.keys) and np.array_equal(t, cv.ticks) and np.array_equal(h, cv.hits_e)):
            bad.append("final LRU differs")
        if not np.array_equal(cache.eviction_log_array(), np.asarray(cv.evictions, np.uint64)):
            bad.append("eviction log differs")
        sk, sv = cache.sketch_arrays()
        if not (np.array_equal(sk, cv.sk_keys) and np.array_equal(sv, cv.sk_vals)):
            bad.append("sketch differs")
        row = dict(batch=n_batches - 1, depth=depth, dyn=rk._step.scalars(0).get("dyn"), bad=bad)
        log(row)
        return [row], dict(rk=rk, cache=cache, dep=dep)
    for i in range(n_batches):
        hb = gen.next()
        idx = torch.from_numpy(hb.indices).cuda()
        offs = torch.from_numpy(hb.offsets).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out, cnt = rk.execute_csr(idx, offs, hb.feature_tables, hb.feature_ops, B, batch_id=i)
        torch.cuda.synchronize()
        t_gpu = time.perf_counter() - t0
        keys, lens = keys_sample_major(hb.indices, hb.offsets, hb.feature_tables, B)
        t0 = time.perf_counter()
        pv.run(keys, lens, B, i)
        t_cpu = time.perf_counter() - t0
        mg, mo = rk.batch_metrics[-1], pv.metrics[-1]
        bad = []
        for a, b in (("cache_hits", "hits"), ("cache_misses", "misses"), ("pushdown_groups", "pushdown_groups"),
                     ("pushdown_rows", "pushdown_rows"), ("raw_rows", "raw_rows")):
            if getattr(mg, a) != mo[b]:
                bad.append(f"{a} {getattr(mg, a)} != {mo[b]}")
        k, t, h = cache.lru_arrays()
        if not (np.array_equal(k, cv.keys) and np.array_equal(t, cv.ticks) and np.array_equal(h, cv.hits_e)):
            n = min(len(k), len(cv.keys))
            first = int(np.nonzero((k[:n] != cv.keys[:n]) | (t[:n] != cv.ticks[:n]))[0][:1].tolist()[0]) \
                if n and ((k[:n] != cv.keys[:n]) | (t[:n] != cv.ticks[:n])).any() else -1
            bad.append(f"LRU differs: {len(k)} vs {len(cv.keys)} entries, first diff at {first}")
        ev = cache.eviction_log_array()
        if not np.array_equal(ev, np.asarray(cv.evictions, np.uint64)):
            bad.append(f"eviction log differs: {len(ev)} vs {len(cv.evictions)}")
        sk, sv = cache.sketch_arrays()
        if not (np.array_equal(sk, cv.sk_keys) and np.array_equal(sv, cv.sk_vals)):
            bad.append(f"sketch differs: {len(sk)} vs {len(cv.sk_keys)} keys")
        pend = [int(x) for x in _pending_u64(cache)]
        if pend != [int(x) for x in cv.pending]:
            bad.append(f"pending differs: {len(pend)} vs {len(cv.pending)}")
        if check_vectors:
            outh = out.cpu().numpy()
            F = len(hb.feature_tables)
            for _ in range(check_vectors):
                f, s_ = int(rng.integers(F)), int(rng.integers(B))
                b = f * B + s_
                ix = hb.indices[hb.offsets[b]:hb.offsets[b + 1]]
                ref = O.pool_flat(O.rows_of(0, f, D, ix), hb.feature_ops[f])
                got = outh[s_, f * D:(f + 1) * D]
                if ref.tobytes() != got.tobytes():
                    bad.append(f"pooled bag (s={s_}, f={f}) not bit-identical to flat "
                               f"(ratio {O.tolerance_ratio(ref, got):.3g})")
                    break
        row = dict(batch=i, hits=mg.cache_hits, misses=mg.cache_misses, hit_rate=mg.hit_rate,
                   offers=mo["n_offers"], accepted=mo["n_accepted"], entries=len(cv), gpu_s=round(t_gpu, 4),
                   cpu_s=round(t_cpu, 3), latency_ms=round(mg.latency * 1e3, 3), bad=bad)
        log(row)
        report.append(row)
    return report, dict(rk=rk, cache=cache, dep=dep)


def _pending_u64(cache):
    import ctypes
    n_p = cache._scalars()["pending"]
    cap = max(1, n_p)
    out = torch.empty(cap, dtype=torch.int64, device=cache.device)
    n = ctypes.c_int64(0)
    cache._L.fx_cache_pending(cache._h, out.data_ptr(), cap, ctypes.byref(n), 0)
    torch.cuda.synchronize()
    return out[:n.value].cpu().numpy().view(np.uint64)
