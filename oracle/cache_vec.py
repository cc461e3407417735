"""Vectorised canonical-order row cache (TEST INFRASTRUCTURE ONLY).

A numpy restatement of the reference AdaptiveCache + FrequencySketch
(cache.py:114-352) driven in the canonical per-batch order of Ranker
(ranker.py:218-442), for ROW keys of one size S. It is the
same algorithm as `restate.CacheOracle` + `restate.PipelineOracle`, but
batched with np.unique / searchsorted so that a cfg3-sized batch (32 tables,
2.6 M probes) runs in about a second instead of minutes:

  apply_pending_admissions (cache.py:344-352)
  -> probe every occurrence in (lookup, feature, position) order
     (cache.py:189-202): a key present at batch start hits on every
     occurrence (nothing is inserted mid-batch), its last_tick becomes
     tick0 + (ordinal of its last occurrence) + 1 and its hits grow by its
     multiplicity; a missing key bumps the sketch by its multiplicity
  -> offers of raw-fetched misses in first raw-occurrence order
     (ranker.py:338-340, 417-423; cache.py:237-268) — the only sequential
     loop, over candidate estimates only
  -> record -> propose -> resize -> stage_hot_admissions(limit) -> age
     (ranker.py:425-442; cache.py:290-342, 128-136).

Checked against restate.CacheOracle (itself pinned to the reference's own
sessions in tests/golden) by tests/test_cache_vec.py. Keys are the u64
encoding table << 40 | row; their numeric order equals the reference's
(table, row) tuple order, which `hottest` sorts by (cache.py:138-143).
"""

from __future__ import annotations

import numpy as np

U64 = np.uint64


class RowCacheVec:
    def __init__(self, budget_bytes: int, row_bytes: int, admission: str = "sketch", decay: float = 0.5,
                 prune: float = 0.25, record_evictions: bool = False):
        self.budget = int(budget_bytes)
        self.S = int(row_bytes)
        self.admission = admission
        self.decay, self.prune = decay, prune
        self.keys = np.zeros(0, U64)        # LRU order (ascending last_tick)
        self.ticks = np.zeros(0, np.int64)
        self.hits_e = np.zeros(0, np.int64)
        self.sk_keys = np.zeros(0, U64)     # sorted
        self.sk_vals = np.zeros(0, np.float64)
        self.pending: list = []
        self.tick = 0
        self.hits = 0
        self.misses = 0
        self.evictions: list | None = [] if record_evictions else None

    # ---------------------------------------------------------------- helpers
    @property
    def used(self) -> int:
        return int(self.keys.size) * self.S

    def __len__(self):
        return int(self.keys.size)

    def _member(self, q: np.ndarray) -> np.ndarray:
        if self.keys.size == 0:
            return np.zeros(q.size, bool)
        srt = np.sort(self.keys)
        p = np.searchsorted(srt, q)
        p[p >= srt.size] = 0
        return srt[p] == q

    def estimate(self, q: np.ndarray) -> np.ndarray:
        """FrequencySketch.estimate (cache.py:125-126), 0.0 for absent keys."""
        q = np.asarray(q, U64)
        out = np.zeros(q.size, np.float64)
        if self.sk_keys.size == 0 or q.size == 0:
            return out
        p = np.searchsorted(self.sk_keys, q)
        p[p >= self.sk_keys.size] = 0
        m = self.sk_keys[p] == q
        out[m] = self.sk_vals[p[m]]
        return out

    def _bump(self, k: np.ndarray, w: np.ndarray):
        """sketch.bump(key, weight) for distinct keys (cache.py:122-123)."""
        if k.size == 0:
            return
        allk = np.concatenate([self.sk_keys, k])
        allv = np.concatenate([self.sk_vals, w.astype(np.float64)])
        u, inv = np.unique(allk, return_inverse=True)
        v = np.zeros(u.size, np.float64)
        # existing value first, then + weight: one addition per key, exact
        np.add.at(v, inv[:self.sk_keys.size], allv[:self.sk_keys.size])
        np.add.at(v, inv[self.sk_keys.size:], allv[self.sk_keys.size:])
        self.sk_keys, self.sk_vals = u, v

    def _evict_head(self, n: int):
        if n <= 0:
            return
        if n > self.keys.size:
            raise KeyError("popitem(): dictionary is empty")  # the reference's OrderedDict
        if self.evictions is not None:
            self.evictions.extend(int(x) for x in self.keys[:n])
        self.keys, self.ticks, self.hits_e = self.keys[n:], self.ticks[n:], self.hits_e[n:]

    def _append(self, k: np.ndarray, t: np.ndarray):
        self.keys = np.concatenate([self.keys, np.asarray(k, U64)])
        self.ticks = np.concatenate([self.ticks, np.asarray(t, np.int64)])
        self.hits_e = np.concatenate([self.hits_e, np.zeros(len(k), np.int64)])

    # ---------------------------------------------------------------- steps
    def apply_pending(self) -> int:
        """cache.py:344-352: install staged keys, always-admit _insert."""
        n = 0
        for key in self.pending:
            if self._member(np.array([key], U64))[0]:
                continue
            if self.S > self.budget:
                continue
            over = (self.keys.size + 1) * self.S - self.budget
            self._evict_head(max(0, -(-over // self.S)))
            self.tick += 1
            self._append([key], [self.tick])
            n += 1
        self.pending = []
        return n

    def probe(self, keys_sm: np.ndarray):
        """Probe every occurrence (sample-major order). Returns
        (uniq, first_ord, last_ord, mult, hit, inverse)."""
        keys_sm = np.asarray(keys_sm, U64)
        nnz = keys_sm.size
        tick0 = self.tick
        if nnz == 0:
            z = np.zeros(0, np.int64)
            return np.zeros(0, U64), z, z, z, np.zeros(0, bool), z
        uniq, first, inv, cnt = np.unique(keys_sm, return_index=True, return_inverse=True, return_counts=True)
        inv = inv.reshape(-1)
        last = np.zeros(uniq.size, np.int64)
        np.maximum.at(last, inv, np.arange(nnz, dtype=np.int64))
        hit = self._member(uniq)
        if hit.any():
            hk = uniq[hit]
            # existing entries that were hit: drop from their LRU position,
            # re-append in last-occurrence order with their new ticks
            order = np.argsort(self.keys, kind="stable")
            pos = order[np.searchsorted(self.keys[order], hk)]
            old_hits = self.hits_e[pos]
            keep = np.ones(self.keys.size, bool)
            keep[pos] = False
            o = np.argsort(last[hit], kind="stable")
            self.keys = np.concatenate([self.keys[keep], hk[o]])
            self.ticks = np.concatenate([self.ticks[keep], tick0 + last[hit][o] + 1])
            self.hits_e = np.concatenate([self.hits_e[keep], (old_hits + cnt[hit])[o]])
        self._bump(uniq[~hit], cnt[~hit])
        self.tick += nnz
        self.hits += int(cnt[hit].sum())
        self.misses += int(cnt[~hit].sum())
        return uniq, first.astype(np.int64), last, cnt.astype(np.int64), hit, inv

    def offer_many(self, cand: np.ndarray) -> np.ndarray:
        """offer(key) for each distinct candidate in order (cache.py:237-268).
        A candidate cached when its turn comes returns True with no side
        effect; one that an earlier offer of the same call evicted is absent
        again and goes through admission (possible when several batches are
        in flight). Returns the accept mask."""
        cand = np.asarray(cand, U64)
        n = cand.size
        acc = np.zeros(n, bool)
        if n == 0:
            return acc
        S, budget = self.S, self.budget
        c_est = self.estimate(cand).tolist()
        v_est = self.estimate(self.keys).tolist() if self.admission == "sketch" else []
        vpos = {k: i for i, k in enumerate(self.keys.tolist())}   # initial entries' LRU positions
        e = self.keys.size           # live entries
        h = 0                        # LRU head position in V = [entries] ++ [accepts]
        acc_idx = []
        sketch = self.admission == "sketch"
        for j, k in enumerate(cand.tolist()):
            p = vpos.get(k)
            if p is not None and p >= h:   # still cached: offer -> True
                acc[j] = True
                continue
            if S > budget:
                continue
            if (e + 1) * S > budget:
                if sketch:
                    ve = v_est[h] if h < len(v_est) else c_est[acc_idx[h - len(v_est)]]
                    if c_est[j] < ve:
                        continue
                while (e + 1) * S > budget:
                    if e == 0:
                        raise KeyError("popitem(): dictionary is empty")
                    h += 1
                    e -= 1
            acc[j] = True
            acc_idx.append(j)
            e += 1
        n_exist = self.keys.size
        n_acc = len(acc_idx)
        ev_exist = min(h, n_exist)
        ev_acc = h - ev_exist          # accepted in this call and evicted again
        if self.evictions is not None:
            self.evictions.extend(int(x) for x in self.keys[:ev_exist])
            self.evictions.extend(int(x) for x in cand[acc_idx[:ev_acc]])
        t = self.tick + 1 + np.arange(n_acc, dtype=np.int64)
        self.keys = np.concatenate([self.keys[ev_exist:], cand[acc_idx[ev_acc:]]])
        self.ticks = np.concatenate([self.ticks[ev_exist:], t[ev_acc:]])
        self.hits_e = np.concatenate([self.hits_e[ev_exist:], np.zeros(n_acc - ev_acc, np.int64)])
        self.tick += n_acc
        return acc

    def resize(self, new_budget: int, fetch: bool = True):
        """cache.py:290-309 (row sizes known: every row is S bytes)."""
        grow = new_budget > self.budget
        self.budget = int(new_budget)
        over = self.used - self.budget
        if over > 0:
            self._evict_head(-(-over // self.S))
        if grow and fetch:
            self.stage(None)

    def stage(self, limit):
        """stage_hot_admissions (cache.py:311-342): hottest sketch keys by
        (-count, key), skipping cached / pending keys and keys that do not
        fit the spare room."""
        room = self.budget - self.used
        if room <= 0 or self.sk_keys.size == 0:
            return []
        order = np.lexsort((self.sk_keys, -self.sk_vals))
        if limit is not None:
            order = order[:limit]
        ranked = self.sk_keys[order]
        excl = self._member(ranked) | np.isin(ranked, np.asarray(self.pending, U64))
        staged = []
        for k, x in zip(ranked.tolist(), excl.tolist()):
            if x or self.S > room:
                continue
            self.pending.append(k)
            staged.append(k)
            room -= self.S
            if limit is not None and len(staged) >= limit:
                break
        return staged

    def age(self):
        """cache.py:128-136."""
        v = self.sk_vals * self.decay
        keep = v >= self.prune
        self.sk_keys, self.sk_vals = self.sk_keys[keep], v[keep]


class RowPipelineVec:
    """Canonical per-batch order of Ranker (ranker.py:218-442) on one server
    with a row cache of one row size: the PipelineOracle restricted to what
    the cfg3 workload exercises (single shard per table, uniform dims).
    `threshold` None: every miss is raw-fetched and offered; an int t >= 2:
    a bag's misses are pushed down when there are >= t of them (one server,
    so a bag is one group, pooling.py:88-100) and only raw misses are
    offered. `policy`/`tracker` follow restate.CachePolicyO/LoadTrackerO."""

    def __init__(self, cache: RowCacheVec, threshold=None, policy=None, tracker=None, adaptive=True,
                 admit_per_batch=64):
        self.cache = cache
        self.threshold = threshold
        self.policy, self.tracker = policy, tracker
        self.adaptive, self.admit = adaptive, admit_per_batch
        self.metrics = []

    def run(self, keys_sm: np.ndarray, bag_len_sm: np.ndarray, n_lookups: int, batch_id: int = 0):
        return self.finish(self.start(keys_sm, bag_len_sm, n_lookups, batch_id))

    def start(self, keys_sm: np.ndarray, bag_len_sm: np.ndarray, n_lookups: int, batch_id: int = 0):
        """_start_batch (ranker.py:218-257): apply_pending -> admission check
        -> probes -> plan. Returns the in-flight batch state."""
        c = self.cache
        keys_sm = np.asarray(keys_sm, U64)
        c.apply_pending()
        if self.policy is not None:
            m = self.policy.m
            need = m.fixed + n_lookups * m.per
            if need > m.cap:
                raise OverflowError("nn capacity")
            if need + c.budget > m.cap:
                if not self.adaptive:
                    raise OverflowError("fixed cache")
                c.resize(m.target(n_lookups), fetch=False)
        uniq, first, last, mult, hit, inv = c.probe(keys_sm)
        hit_occ = hit[inv] if keys_sm.size else np.zeros(0, bool)
        nb = bag_len_sm.size
        bag_of = np.repeat(np.arange(nb), bag_len_sm)
        miss_per_bag = np.bincount(bag_of, weights=~hit_occ, minlength=nb).astype(np.int64)
        if self.threshold is None:
            push_bag = np.zeros(nb, bool)
        else:
            push_bag = miss_per_bag >= self.threshold
        raw_occ = ~hit_occ & ~push_bag[bag_of]
        # first raw occurrence of each key, in sample-major ordinal order
        ords = np.nonzero(raw_occ)[0]
        ku, kfirst = np.unique(inv[ords], return_index=True)
        cand_u = ku[np.argsort(ords[kfirst], kind="stable")]
        hits = int(mult[hit].sum())
        nnz = int(keys_sm.size)
        return dict(batch_id=batch_id, size=n_lookups, cand=uniq[cand_u], uniq=uniq, hit=hit, mult=mult,
                    hit_occ=hit_occ, hits=hits, misses=nnz - hits,
                    pushdown_groups=int(push_bag[miss_per_bag > 0].sum()),
                    pushdown_rows=int(miss_per_bag[push_bag].sum()), raw_rows=int(raw_occ.sum()),
                    subrequests=int((miss_per_bag > 0).sum()))

    def finish(self, st):
        """_finish_batch (ranker.py:364-442): offers of the raw-fetched rows in
        first raw-occurrence order — a key installed since the probes (a later
        batch's apply_pending, pipeline_depth > 1) is present: offer() -> True
        with no side effect — then maintenance."""
        c = self.cache
        cand = st["cand"]
        accepted = c.offer_many(cand)
        level = None
        staged = []
        if self.tracker is not None and self.policy is not None:
            level = self.tracker.record(st["size"])
            if self.adaptive:
                prop = self.policy.propose(c.budget, level, self.tracker.value())
                if prop != c.budget:
                    c.resize(prop, fetch=True)
                if self.admit > 0:
                    staged = c.stage(self.admit)
                c.age()
        self.metrics.append(dict(batch_id=st["batch_id"], size=st["size"], hits=st["hits"], misses=st["misses"],
                                 pushdown_groups=st["pushdown_groups"], pushdown_rows=st["pushdown_rows"],
                                 raw_rows=st["raw_rows"], subrequests=st["subrequests"], load_level=level,
                                 n_offers=int(cand.size), n_accepted=int(accepted.sum()), staged=staged,
                                 budget=c.budget if len(c) else None, used=c.used if len(c) else None))
        return dict(uniq=st["uniq"], hit=st["hit"], mult=st["mult"], cand=cand, accepted=accepted,
                    hit_occ=st["hit_occ"])

    def run_trace(self, batches, depth: int = 1):
        """Closed-loop replay with `depth` batches in flight (ranker.py:161-182):
        S0..S(d-1) F0 Sd F1 ... ; batches = [(keys_sm, bag_len_sm, n_lookups, id)]."""
        inflight = []
        for b in batches:
            inflight.append(self.start(*b))
            if len(inflight) >= depth:
                self.finish(inflight.pop(0))
        while inflight:
            self.finish(inflight.pop(0))


def keys_sample_major(indices: np.ndarray, offsets: np.ndarray, feature_tables, batch_size: int):
    """Table-major CSR (bag = f*B + s) -> (u64 keys in (sample, feature,
    position) order, bag lengths in sample-major order)."""
    F, B = len(feature_tables), batch_size
    lens_tm = np.diff(offsets).reshape(F, B)
    lens_sm = lens_tm.T.reshape(-1)
    tab = np.repeat(np.asarray(feature_tables, np.uint64), B)            # per tm bag
    key_tm = (np.repeat(tab, lens_tm.reshape(-1)) << U64(40)) | np.asarray(indices, np.int64).astype(U64)
    # gather in sample-major bag order
    sm_bags = (np.arange(F)[None, :] * B + np.arange(B)[:, None]).reshape(-1)
    starts = offsets[:-1][sm_bags]
    ln = lens_tm.reshape(-1)[sm_bags]
    pos = np.repeat(starts, ln) + (np.arange(int(ln.sum())) - np.repeat(np.cumsum(ln) - ln, ln))
    return key_tm[pos], lens_sm.astype(np.int64)
