"""Pin the CPU oracle (oracle/restate.py) against golden vectors produced by
the reference embserve package itself (tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

import oracle as O


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def test_prf_table_block_bit_exact(golden_dir):
    z = _load(golden_dir, "prf.npz")
    i = 0
    while f"case{i}" in z:
        seed, t, d, s, e = (int(v) for v in z[f"case{i}"])
        got = O.table_block(seed, t, d, s, e)
        assert got.tobytes() == z[f"block{i}"].tobytes(), i
        i += 1
    rows = O.rows_of(3, 2, 64, [0, 1, 77, 99_999])
    assert rows.tobytes() == z["rowv"].tobytes()


def test_prf_value_range_includes_one():
    # store.py:88-89: (1 - 2^-52)*2 - 1 rounds to exactly 1.0f
    assert np.float32(((2**53 - 1) * 2.0**-53) * 2.0 - 1.0) == np.float32(1.0)


def test_partial_pool_bit_exact(golden_dir):
    z = _load(golden_dir, "pool.npz")
    for k in range(int(z["n_pp"][0])):
        seed, rows, dim = (int(v) for v in z[f"pp{k}_meta"])
        idx = z[f"pp{k}_idx"]
        raw = O.rows_of(seed, 0, dim, idx)
        assert raw.tobytes() == z[f"pp{k}_raw"].tobytes()
        got = O.seq_sum_f64(raw).astype(np.float32)
        assert got.tobytes() == z[f"pp{k}_vec"].tobytes()


def test_combine_and_flat_bit_exact(golden_dir):
    z = _load(golden_dir, "pool.npz")
    for k in range(int(z["n_c"][0])):
        rows = z[f"c{k}_rows"]
        owners = z[f"c{k}_owner"]
        pushed = set(int(g) for g in z[f"c{k}_pushed"])
        op = "sum" if int(z[f"c{k}_op"][0]) == 0 else "mean"
        partials, raw_pos = [], []
        for g in np.unique(owners):
            mem = np.nonzero(owners == g)[0]
            if int(g) in pushed:
                partials.append((O.seq_sum_f64(rows[mem]).astype(np.float32), len(mem), int(g)))
            else:
                raw_pos.extend(mem.tolist())
        raw = [rows[i] for i in sorted(raw_pos)]
        assert O.combine_partials(partials, raw, op).tobytes() == z[f"c{k}_comb"].tobytes()
        assert O.pool_flat(rows, op).tobytes() == z[f"c{k}_flat"].tobytes()
        if np.abs(rows).max() <= 1.0:  # the reference's property holds for rows in [-1, 1]
            assert O.within_tolerance(z[f"c{k}_flat"], z[f"c{k}_comb"])
    ex = O.combine_partials([(np.array([1.5], np.float32), 1, 1), (np.array([1e8], np.float32), 1, 2),
                             (np.array([-1e8], np.float32), 1, 0)], [], "sum")
    assert ex.tobytes() == z["order_example"].tobytes()


def test_routing_golden(golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "routing.json")))
    for c in cases:
        pl = O.Placement.from_specs({0: c["num_rows"]}, [tuple(s) for s in c["placement"]])
        assert O.resolve_many(pl, 0, c["idx"]).tolist() == c["servers"]
        groups = O.group_feature(pl, 0, c["feature"])
        assert [[g[0], g[1], g[2]] for g in groups] == c["groups"]


def test_zipf_golden(golden_dir):
    z = _load(golden_dir, "zipf.npz")
    for i in range(4):
        n, a, seed, k = z[f"meta{i}"]
        got = O.ZipfSampler(int(n), float(a)).sample(np.random.default_rng(int(seed)), int(k))
        assert np.array_equal(got, z[f"s{i}"])


def test_dedup_matches_numpy_unique():
    rng = np.random.default_rng(0)
    t = rng.integers(0, 26, size=5000)
    r = rng.integers(0, 1000, size=5000)
    keys = O.make_keys(t, r)
    u, inv, cnt = O.dedup_keys(keys)
    assert np.array_equal(u[inv], keys)
    assert cnt.sum() == keys.size


def test_cache_sessions_golden(golden_dir):
    sessions = json.load(open(os.path.join(golden_dir, "cache.json")))
    for s in sessions:
        rb = s["row_bytes"]
        c = O.CacheOracle(s["budget0"], admission=s["admission"])
        for st in s["steps"]:
            c.apply_pending()
            hits = [c.get(tuple(k)) for k in st["keys"]]
            assert hits == st["hits"]
            offered = [c.offer(tuple(k), rb) for k in st["offers"]]
            assert offered == st["offered"]
            if st["op"] is not None:
                c.resize(st["op"][1], lambda t: rb, fetch=True)
            staged = c.stage(lambda t: rb, 8)
            assert [list(k) for k in staged] == st["staged"]
            c.age()
            assert [list(k) for k in c.lru_keys()] == st["lru"]
            assert [c.entries[tuple(k)][0] for k in st["lru"]] == st["ticks"]
            assert (c.budget, c.used, c.tick) == (st["budget"], st["used"], st["tick"])
            assert sorted([[k[0], k[1], v] for k, v in c.sketch.items()]) == st["sketch"]
        assert [list(k) for k in c.evictions] == s["evictions"]


def _pipeline_for(rec):
    dims = {m[0]: m[2] for m in rec["metas"]}
    pl = O.Placement.from_specs({m[0]: m[1] for m in rec["metas"]}, [tuple(p) for p in rec["placement"]])
    cache = policy = tracker = None
    if "cache" in rec:
        cc = rec["cache"]
        cache = O.CacheOracle(cc["budget"], admission=cc["admission"])
        policy = O.CachePolicyO(O.MemoryModelO(*cc["model"]), cc["hyst"])
        w, hi, lo = cc["tracker"]
        tracker = O.LoadTrackerO(w, hi, lo)
    return O.PipelineOracle(0, dims, pl, threshold=rec["threshold"], cache=cache, policy=policy,
                            tracker=tracker, admit_per_batch=rec.get("cache", {}).get("admit", 64)), pl


@pytest.mark.parametrize("which", [0, 1, 2])
def test_pipeline_oracle_vs_reference_ranker(golden_dir, which):
    recs = json.load(open(os.path.join(golden_dir, "ranker.json")))
    rec = recs[which]
    po, pl = _pipeline_for(rec)
    # the reference's cache budget at batch start is recorded before run
    for bi, lookups in enumerate(rec["batches"]):
        bb = O.bag_batch_from_lists([[(t, op, ix) for t, op, ix in lk] for lk in lookups], batch_id=bi)
        vecs, counters, _ = po.run(bb)
        m = po.metrics[-1]
        ref_m = rec["metrics"][bi]
        for key in ("hits", "misses", "pushdown_groups", "pushdown_rows", "raw_rows"):
            assert m[key] == ref_m[key], (bi, key)
        # per-lookup counters and vectors (bags are created in sample-major order)
        b = 0
        for li, lk in enumerate(lookups):
            agg = [0, 0, 0, 0]
            for fp in range(len(lk)):
                c = counters[b]
                for q in range(4):
                    agg[q] += c[q]
                ref_bits = np.array(rec["results"][bi][li][fp], dtype=np.uint32).view(np.float32)
                # hierarchical combine reproduces the reference bit-exactly
                assert vecs[b].tobytes() == ref_bits.tobytes(), (bi, li, fp)
                b += 1
            assert agg == rec["counters"][bi][li]
        if po.cache is not None:
            assert [list(k) for k in po.cache.lru_keys()] == rec["per_batch_lru"][bi], bi
    if po.cache is not None:
        assert [list(k) for k in po.cache.evictions] == rec["evictions"]
        assert sorted([[k[0], k[1], v] for k, v in po.cache.sketch.items()]) == rec["final_sketch"]


def _kj(k):
    if isinstance(k, tuple) and len(k) == 4 and k[0] == "pooled":
        return ["pooled", k[1], k[2], list(k[3])]
    return list(k)


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_pipeline_oracle_pooled_keyspace_vs_reference(golden_dir, which):
    """Pooled-result keyspace (cache.py:204-223, ranker.py:238-249,401-414):
    per-batch vectors, counters, metrics, LRU (row + pooled keys), used bytes
    (including the bytes leaked by in-place re-puts) and the eviction log."""
    rec = json.load(open(os.path.join(golden_dir, "pooled.json")))["ranker"][which]
    po, _ = _pipeline_for(rec)
    po.cache.pooled = True
    for bi, lookups in enumerate(rec["batches"]):
        bb = O.bag_batch_from_lists([[(t, op, ix) for t, op, ix in lk] for lk in lookups], batch_id=bi)
        vecs, counters, _ = po.run(bb)
        m, ref_m = po.metrics[-1], rec["metrics"][bi]
        for key in ("hits", "misses", "pushdown_groups", "pushdown_rows", "raw_rows"):
            assert m[key] == ref_m[key], (bi, key)
        b = 0
        for li, lk in enumerate(lookups):
            agg = [0, 0, 0, 0]
            for fp in range(len(lk)):
                for q in range(4):
                    agg[q] += counters[b][q]
                ref_bits = np.array(rec["results"][bi][li][fp], dtype=np.uint32).view(np.float32)
                assert vecs[b].tobytes() == ref_bits.tobytes(), (bi, li, fp)
                b += 1
            assert agg == rec["counters"][bi][li]
        assert [_kj(k) for k in po.cache.lru_keys()] == rec["per_batch_lru"][bi], bi
        assert po.cache.used == rec["per_batch_used"][bi]
    assert [_kj(k) for k in po.cache.evictions] == rec["evictions"]


def test_cache_oracle_pooled_api(golden_dir):
    api = json.load(open(os.path.join(golden_dir, "pooled.json")))["api"]
    c = O.CacheOracle(3 * 64, pooled=True)
    v = lambda x: np.full(16, x, np.float32)
    c.pooled_put(("pooled", 0, "sum", (1, 2)), v(9.0))
    c.offer((0, 5), 64)
    c.pooled_put(("pooled", 0, "sum", (1, 2)), v(7.0))
    got = c.pooled_get(("pooled", 0, "sum", (1, 2)))
    c.pooled_put(("pooled", 1, "mean", (3,)), v(4.0))
    assert [_kj(k) for k in c.lru_keys()] == api["lru"]
    assert (c.used, c.tick) == (api["used"], api["tick"])
    assert [float(x) for x in got] == api["got"]
    assert [_kj(k) for k in c.evictions] == api["evictions"]


def test_pooled_fingerprint_is_a_multiset_key():
    a = O.pooled_fingerprint(3, "sum", [5, 1, 5, 9])
    assert a == O.pooled_fingerprint(3, "sum", [9, 5, 1, 5])
    assert a != O.pooled_fingerprint(3, "sum", [5, 1, 9])
    assert a != O.pooled_fingerprint(3, "mean", [5, 1, 5, 9])
    assert a != O.pooled_fingerprint(4, "sum", [5, 1, 5, 9])
    assert a[0] >> 63 == 1
