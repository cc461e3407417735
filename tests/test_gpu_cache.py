"""GPU hot-row cache (K3/K6) vs the reference's AdaptiveCache: scripted
sessions recorded from the reference (tests/golden/cache.json) must replay
bit-exactly — hits, offer decisions, staged keys, LRU order and ticks,
budget/used/tick scalars, sketch contents, eviction log — plus the
reference's own cache unit examples (test_cache.py / acceptance criterion 9)."""

import json
import os
from collections import OrderedDict

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROW_BYTES = 16


@pytest.fixture(scope="module")
def C():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_12794_b200 import cache as C
    return C


def vec(dim=4, fill=1.0):
    return np.full(dim, fill, dtype=np.float32)


def _probe_batch(C, cache, keys):
    """Probe an ordered key list through the batched (dedup) path: unique
    keys, multiplicities and last-occurrence ordinals."""
    dev = cache.device
    first = OrderedDict()
    for i, k in enumerate(keys):
        e = first.setdefault(k, [0, 0])
        e[0] += 1
        e[1] = i
    u = C._u64([C.encode_key(*k) for k in first]).to(dev)
    mult = torch.tensor([v[0] for v in first.values()], dtype=torch.int32, device=dev)
    last = torch.tensor([v[1] for v in first.values()], dtype=torch.int64, device=dev)
    slot = torch.empty(len(first), dtype=torch.int32, device=dev)
    cache.probe_unique(u, mult, last, None, len(keys), slot, n_uniq_host=len(first))
    hit = dict(zip(first, (slot.cpu().numpy() >= 0)))
    return [bool(hit[k]) for k in keys]


@pytest.mark.parametrize("batched", [True, False])
def test_cache_sessions_replay_golden(C, golden_dir, batched):
    sessions = json.load(open(os.path.join(golden_dir, "cache.json")))
    for s in sessions:
        rb = s["row_bytes"]
        cache = C.AdaptiveCache(s["budget0"], admission=s["admission"], record_evictions=True, max_dim=4)
        cache.set_row_bytes(0, rb)
        cache.set_row_bytes(1, rb)
        fetch = lambda t, i: vec()
        for st in s["steps"]:
            cache.apply_pending_admissions()
            keys = [tuple(k) for k in st["keys"]]
            if batched:
                hits = _probe_batch(C, cache, keys)
            else:
                hits = [cache.get(*k) is not None for k in keys]
            assert hits == st["hits"]
            if batched:
                offs = [tuple(k) for k in st["offers"]]
                ones = torch.ones(4, dtype=torch.float32, device=cache.device)
                kk = C._u64([C.encode_key(*k) for k in offs]).to(cache.device)
                src = torch.full((max(len(offs), 1),), ones.data_ptr(), dtype=torch.int64, device=cache.device)
                acc = torch.zeros(max(len(offs), 1), dtype=torch.uint8, device=cache.device)
                cache.offer_keys(kk, len(offs), src, acc)
                offered = [bool(a) for a in acc.cpu().numpy()[:len(offs)]]
            else:
                offered = [cache.offer(k[0], k[1], vec()) for k in st["offers"]]
            assert offered == st["offered"]
            if st["op"] is not None:
                cache.resize(st["op"][1], fetcher=fetch, row_bytes_of=lambda t: rb)
            staged = cache.stage_hot_admissions(fetch, lambda t: rb, limit=8)
            assert [list(k) for k in staged] == st["staged"]
            cache.sketch.age()
            ent = cache.lru_entries()
            assert [list(e[0]) for e in ent] == st["lru"]
            assert [e[1] for e in ent] == st["ticks"]
            assert (cache.budget_bytes, cache.used_bytes, cache.tick) == (st["budget"], st["used"], st["tick"])
            got_sk = sorted([[k[0], k[1], v] for k, v in cache.sketch.ranked()])
            assert got_sk == st["sketch"]
        assert [list(k) for k in cache.eviction_log] == s["evictions"]


def test_lru_eviction_order_example(C):
    cache = C.AdaptiveCache(budget_bytes=3 * ROW_BYTES, admission="always", record_evictions=True, max_dim=4)
    for i in range(3):
        cache.offer(0, i, vec())
    cache.get(0, 0)
    cache.resize(2 * ROW_BYTES, fetcher=None)
    assert cache.eviction_log == [(0, 1)]


def test_get_hit_miss_and_values(C):
    cache = C.AdaptiveCache(budget_bytes=10 * ROW_BYTES, max_dim=4)
    assert cache.get(0, 1) is None
    cache.offer(0, 1, vec(fill=3.5))
    got = cache.get(0, 1)
    assert got is not None and np.array_equal(got, vec(fill=3.5))
    assert cache.hits == 1 and cache.misses == 1 and cache.hit_rate() == 0.5


def test_sketch_admission_protects_hot_victims(C):
    cache = C.AdaptiveCache(budget_bytes=1 * ROW_BYTES, admission="sketch", max_dim=4)
    for _ in range(5):
        cache.get(0, 1)
    cache.offer(0, 1, vec())
    cache.get(0, 2)
    assert cache.offer(0, 2, vec()) is False
    assert cache.contains(0, 1)
    for _ in range(9):
        cache.get(0, 3)
    assert cache.offer(0, 3, vec()) is True
    assert cache.contains(0, 3) and not cache.contains(0, 1)


def test_resize_grow_admits_hottest_async(C):
    cache = C.AdaptiveCache(budget_bytes=0, max_dim=4)
    cache.set_row_bytes(0, ROW_BYTES)
    for _ in range(9):
        cache.get(0, 7)
    for _ in range(3):
        cache.get(0, 8)
    rep = cache.resize(1 * ROW_BYTES, fetcher=lambda t, i: vec(fill=float(i)), row_bytes_of=lambda t: ROW_BYTES)
    assert rep.admitted == [(0, 7)]
    assert not cache.contains(0, 7)  # staged, not yet applied
    assert cache.apply_pending_admissions() == 1
    assert cache.contains(0, 7) and not cache.contains(0, 8)
    assert np.array_equal(cache.get(0, 7), vec(fill=7.0))


def test_resize_shrink_reports_evictions(C):
    cache = C.AdaptiveCache(budget_bytes=3 * ROW_BYTES, admission="always", max_dim=4)
    for i in range(3):
        cache.offer(0, i, vec())
    rep = cache.resize(1 * ROW_BYTES, fetcher=None)
    assert rep.evicted == [(0, 0), (0, 1)]
    assert cache.used_bytes <= cache.budget_bytes


def test_budget_safety(C):
    cache = C.AdaptiveCache(budget_bytes=5 * ROW_BYTES, admission="always", max_dim=4)
    for i in range(50):
        cache.offer(0, i, vec())
        assert cache.used_bytes <= cache.budget_bytes
    assert len(cache) == 5


class _OracleLRU:
    def __init__(self, capacity):
        self.capacity = capacity
        self.entries = OrderedDict()
        self.evictions = []

    def access(self, key):
        if key in self.entries:
            self.entries.move_to_end(key)
            return True
        if len(self.entries) >= self.capacity:
            self.evictions.append(self.entries.popitem(last=False)[0])
        self.entries[key] = True
        return False


def test_criterion9_exact_eviction_sequence(C):
    rng = np.random.default_rng(17)
    cap = 64
    cache = C.AdaptiveCache(budget_bytes=cap * ROW_BYTES, admission="always", record_evictions=True, max_dim=4)
    oracle = _OracleLRU(cap)
    for key in rng.integers(0, 500, size=3000):
        key = int(key)
        hit = cache.get(0, key) is not None
        if not hit:
            cache.offer(0, key, vec())
        assert hit == oracle.access(key)
    assert cache.eviction_log == [(0, k) for k in oracle.evictions]


def test_batched_probe_equals_per_occurrence_probe(C):
    """The dedup-based batched probe (one thread per unique key, hit tick =
    tick0 + last ordinal + 1, sketch += multiplicity) reproduces a sequence of
    per-occurrence get() calls exactly."""
    rng = np.random.default_rng(3)
    a = C.AdaptiveCache(budget_bytes=40 * ROW_BYTES, admission="sketch", max_dim=4)
    b = C.AdaptiveCache(budget_bytes=40 * ROW_BYTES, admission="sketch", max_dim=4)
    for c in (a, b):
        c.set_row_bytes(0, ROW_BYTES)
        for i in range(0, 60, 2):
            c.offer(0, i, vec())
    for _ in range(4):
        keys = [(0, int(k)) for k in rng.integers(0, 80, size=200)]
        ha = _probe_batch(C, a, keys)
        hb = [b.get(*k) is not None for k in keys]
        assert ha == hb
        assert a.lru_entries() == b.lru_entries()
        assert a.sketch.ranked() == b.sketch.ranked()
        assert (a.tick, a.hits, a.misses) == (b.tick, b.hits, b.misses)


@pytest.mark.parametrize("admission", ["sketch", "always"])
def test_parallel_offers_equal_sequential_loop(C, admission):
    """The run-parallel ordered-offer kernel (uniform row size) makes exactly
    the decisions of the sequential reference loop: same accepts, LRU order,
    ticks, eviction log and sketch, across fills, steady state, shrinks and
    grow-stage-apply cycles, with windows larger and smaller than the cache."""
    rng = np.random.default_rng(1)
    for cap_rows in (7, 300, 5000):
        caches = []
        for par in (True, False):
            c = C.AdaptiveCache(cap_rows * ROW_BYTES, admission=admission, record_evictions=True, max_dim=4,
                                slot_capacity=4 * cap_rows + 8)
            c.set_row_bytes(0, ROW_BYTES)
            c.set_parallel_offers(par)
            caches.append(c)
        ones = torch.ones(4, dtype=torch.float32, device=caches[0].device)
        for step in range(6):
            keys = [(0, int(k)) for k in rng.zipf(1.3, size=4 * cap_rows) % (20 * cap_rows)]
            for c in caches:
                c.apply_pending_admissions()
                _probe_batch(C, c, keys)
            # offers: distinct misses in first-occurrence order (some present keys mixed in)
            seen = list(dict.fromkeys(keys))
            accs = []
            for c in caches:
                kk = C._u64([C.encode_key(*k) for k in seen]).to(c.device)
                src = torch.full((len(seen),), ones.data_ptr(), dtype=torch.int64, device=c.device)
                acc = torch.zeros(len(seen), dtype=torch.uint8, device=c.device)
                c.offer_keys(kk, len(seen), src, acc)
                accs.append(acc.cpu().numpy())
            assert np.array_equal(accs[0], accs[1])
            if step == 3:
                for c in caches:
                    c.resize(int(cap_rows * 0.6) * ROW_BYTES, fetcher=None)
            if step == 4:
                for c in caches:
                    c.resize(cap_rows * ROW_BYTES, fetcher=lambda t, i: vec(), row_bytes_of=lambda t: ROW_BYTES)
            for c in caches:
                c.stage_hot_admissions(lambda t, i: vec(), lambda t: ROW_BYTES, limit=16)
                c.sketch.age()
            a, b = caches
            assert a.lru_entries() == b.lru_entries(), (cap_rows, step)
            assert (a.used_bytes, a.tick, a.hits, a.misses) == (b.used_bytes, b.tick, b.hits, b.misses)
            assert a.sketch.ranked() == b.sketch.ranked()
        assert caches[0].eviction_log == caches[1].eviction_log


@pytest.mark.parametrize("thr", [None, 2])
def test_ranker_large_cache_vs_oracle(thr):
    """A cache much larger than each batch's offers (the partial LRU-order
    path: only the oldest entries that can be evicted are ordered) against
    the canonical-order oracle: per-batch metrics, LRU order and evictions."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle as O
    import paper_2410_12794_b200 as P
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen
    rows, D, B = (60_000, 40_000, 60_000, 9_000), 16, 64
    metas = [P.TableMeta(t, n, D) for t, n in enumerate(rows)]
    placement = [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(rows)]
    dep = P.init_store(metas, placement, 0)
    budget = 8_000 * D * 4
    model = (budget + 1000 + B, 1000, 1)
    cache = C.AdaptiveCache(budget, admission="sketch", record_evictions=True, max_dim=D)
    rk = Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=thr, admit_per_batch=64),
                cache=cache, policy=C.CachePolicy(C.MemoryModel(*model)), tracker=C.LoadTracker(4, 10 ** 9, 0))
    pl = O.Placement.from_specs({m.table_id: m.num_rows for m in metas},
                                [(s.table_id, s.start, s.end, s.server_id) for s in placement])
    oc = O.CacheOracle(budget, admission="sketch")
    po = O.PipelineOracle(0, {m.table_id: D for m in metas}, pl, threshold=thr, cache=oc,
                          policy=O.CachePolicyO(O.MemoryModelO(*model)), tracker=O.LoadTrackerO(4, 10 ** 9, 0),
                          admit_per_batch=64)
    gen = DlrmBatchGen(rows, 0.9, B, (1, 8), seed=5)
    F = len(rows)
    for it in range(24):
        hb = gen.next()
        rk.execute_csr(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(), tuple(range(F)),
                       ("sum",) * F, B, batch_id=it)
        bb = O.BagBatch(hb.offsets.astype(np.int64), hb.indices.astype(np.int64), np.repeat(np.arange(F), B),
                        ["sum"] * (F * B), np.tile(np.arange(B), F), np.repeat(np.arange(F), B), B, it)
        po.run(bb)
        m, om = rk.batch_metrics[-1], po.metrics[-1]
        assert (m.cache_hits, m.cache_misses, m.raw_rows) == (om["hits"], om["misses"], om["raw_rows"]), it
        assert rk.cache.lru_keys() == oc.lru_keys(), it
    assert rk.cache.eviction_log == oc.evictions
    if thr is None:  # the cache filled and evicted with most entries outside the sorted prefix
        assert len(oc.evictions) > 0 and len(oc.lru_keys()) > 5_000


def test_cache_frees_device_memory_on_del(C):
    """Dropping the last reference to a cache returns its device buffers at
    once (no cache <-> sketch cycle waiting for a GC pass)."""
    import gc
    torch.cuda.synchronize()
    gc.disable()
    try:
        free0, _ = torch.cuda.mem_get_info()
        cache = C.AdaptiveCache(1 << 30, admission="sketch", max_dim=128, slot_capacity=1 << 21)
        cache.offer(0, 1, np.ones(128, np.float32))
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info()
        assert free0 - free1 >= (1 << 21) * 512  # the row store alone
        del cache
        torch.cuda.synchronize()
        free2, _ = torch.cuda.mem_get_info()
        assert free0 - free2 < 64 << 20, (free0, free1, free2)
    finally:
        gc.enable()
