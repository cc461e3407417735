"""numpy restatement of the reference hot path (test infrastructure only).

Reference paths are relative to /root/reference/pkg/src/embserve.
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "mix64", "table_base", "rows_of", "table_block", "pooled_fingerprint",
    "seq_sum_f64", "pool_flat", "combine_partials", "plan_modes",
    "Placement", "resolve_many", "group_feature",
    "ZipfSampler", "dedup_keys", "make_keys",
    "CacheOracle", "MemoryModelO", "LoadTrackerO", "CachePolicyO",
    "BagBatch", "bag_batch_from_lists", "flat_pool_batch",
    "PipelineOracle", "within_tolerance", "tolerance_ratio",
]

_U64 = np.uint64
_GOLDEN = _U64(0x9E3779B97F4A7C15)
_M1 = _U64(0xBF58476D1CE4E5B9)
_M2 = _U64(0x94D049BB133111EB)

REL_TOL = 1e-5   # ranker.py:472-473
ABS_FLOOR = 1e-6


# ---------------------------------------------------------------- content PRF

def mix64(x) -> np.ndarray:
    """SplitMix64 finaliser over uint64 with wraparound (store.py:62-67)."""
    x = np.asarray(x, dtype=_U64)
    with np.errstate(over="ignore"):
        x = x + _GOLDEN
        x = (x ^ (x >> _U64(30))) * _M1
        x = (x ^ (x >> _U64(27))) * _M2
        return x ^ (x >> _U64(31))


_SALT_A = _U64(0xA0761D6478BD642F)
_SALT_B = _U64(0xE7037ED1A0B428DB)
_OPC = {"sum": 0, "mean": 1}


def pooled_fingerprint(table_id: int, op: str, indices):
    """The B200 cache's identifier (A, B) for the reference's pooled key
    ("pooled", table, op, sorted(indices)) (cache.py:209), restated from
    include/flexemb.h (fx_bag_fingerprint): order-independent sums of
    mix64(x ^ salt), finalised with table, op and L. Used by tests to map the
    reference's tuple keys onto device keys."""
    x = np.asarray(list(indices), dtype=np.int64).view(_U64)
    with np.errstate(over="ignore"):
        sa = _U64(int(mix64(x ^ _SALT_A).sum(dtype=_U64)) if x.size else 0)
        sb = _U64(int(mix64(x ^ _SALT_B).sum(dtype=_U64)) if x.size else 0)
        t = _U64(table_id)
        opc = _U64(_OPC[op])
        L = _U64(x.size)
        a = mix64(sa ^ mix64(mix64(t ^ _SALT_A) + opc) ^ (L * _SALT_B)) | _U64(1 << 63)
        b = mix64(sb ^ mix64(mix64(t ^ _SALT_B) + opc) ^ (L * _SALT_A))
    return int(a), int(b)


def table_base(seed: int, table_id: int) -> np.uint64:
    """base_t = mix64(t ^ mix64(seed)) (store.py:70-74)."""
    s = mix64(np.array([seed], dtype=_U64))
    return mix64(np.array([table_id], dtype=_U64) ^ s)[0]


def rows_of(seed: int, table_id: int, dim: int, rows) -> np.ndarray:
    """Rows `rows` (any order, duplicates allowed) of table `table_id`:
    element (r, c) = f32(((mix64(base + r*dim + c) >> 11) * 2^-53) * 2 - 1)
    (store.py:82-89, restated for arbitrary row sets)."""
    rows = np.asarray(rows, dtype=np.int64).reshape(-1)
    base = table_base(seed, table_id)
    ctr = (rows.astype(_U64)[:, None] * _U64(dim)
           + np.arange(dim, dtype=_U64)[None, :])
    with np.errstate(over="ignore"):
        bits = mix64(ctr + base)
    unit = (bits >> _U64(11)).astype(np.float64) * (1.0 / float(1 << 53))
    return (unit * 2.0 - 1.0).astype(np.float32)


def table_block(seed: int, table_id: int, dim: int, start: int, end: int) -> np.ndarray:
    """(end-start, dim) block (store.py:82-89)."""
    return rows_of(seed, table_id, dim, np.arange(start, end, dtype=np.int64))


# ---------------------------------------------------------------- pooling

def seq_sum_f64(rows: np.ndarray) -> np.ndarray:
    """Element-wise f64 sum of rows in input order (pooling.py:60-71)."""
    rows = np.asarray(rows)
    acc = np.zeros(rows.shape[-1], dtype=np.float64)
    for r in rows:
        acc += r
    return acc


def pool_flat(rows: np.ndarray, op: str) -> np.ndarray:
    """pooling.py:74-85: f64 sequential sum, Mean divides once, emit f32."""
    rows = np.asarray(rows)
    if rows.shape[0] == 0:
        raise ValueError("pool_flat: empty vector list")
    total = seq_sum_f64(rows)
    if op == "mean":
        total = total / rows.shape[0]
    return total.astype(np.float32)


def combine_partials(partials, raw, op: str) -> np.ndarray:
    """pooling.py:103-123. partials: list of (vector f32, count, source);
    folded by ascending source, then raw vectors in given order, f64."""
    if not partials and not raw:
        raise ValueError("combine_partials: nothing to combine")
    ordered = sorted(partials, key=lambda p: p[2])
    vecs = [np.asarray(p[0], np.float32) for p in ordered] + [np.asarray(r, np.float32) for r in raw]
    total = seq_sum_f64(np.stack(vecs))
    if op == "mean":
        total = total / (sum(p[1] for p in partials) + len(raw))
    return total.astype(np.float32)


def plan_modes(group_sizes: dict, threshold):
    """pooling.py:88-100 (threshold None = no pushdown, ranker.py:270-271)."""
    if threshold is None:
        return {k: "raw" for k in group_sizes}
    if threshold < 2:
        raise ValueError(f"pushdown threshold must be >= 2, got {threshold}")
    return {k: ("pushdown" if n >= threshold else "raw") for k, n in group_sizes.items()}


def within_tolerance(ref, got, rel=REL_TOL, floor=ABS_FLOOR) -> bool:
    return tolerance_ratio(ref, got, rel, floor) <= 1.0


def tolerance_ratio(ref, got, rel=REL_TOL, floor=ABS_FLOOR) -> float:
    """max |a-b| / max(floor, rel*|ref|) (ranker.py:487-491)."""
    ref = np.asarray(ref, np.float64)
    got = np.asarray(got, np.float64)
    if ref.size == 0:
        return 0.0
    diff = np.abs(ref - got)
    bound = np.maximum(floor, rel * np.abs(ref))
    return float((diff / bound).max())


# ---------------------------------------------------------------- routing

@dataclass
class Placement:
    """Per table: sorted shard starts, owning server, table rows
    (routing.py:17-21, 100-114)."""
    starts: dict
    servers: dict
    num_rows: dict

    @staticmethod
    def from_specs(metas: dict, specs) -> "Placement":
        """metas: table -> rows; specs: iterable of (table, start, end, server)."""
        starts, servers = {}, {}
        for t in metas:
            sh = sorted((s for s in specs if s[0] == t), key=lambda s: s[1])
            starts[t] = np.array([s[1] for s in sh], dtype=np.int64)
            servers[t] = np.array([s[3] for s in sh], dtype=np.int64)
        return Placement(starts, servers, dict(metas))


def resolve_many(pl: Placement, table_id: int, idx) -> np.ndarray:
    """servers[searchsorted(starts, idx, 'right') - 1] (routing.py:87-97)."""
    idx = np.asarray(idx, dtype=np.int64)
    n = pl.num_rows[table_id]
    if idx.size and (idx.min() < 0 or idx.max() >= n):
        bad = int(idx[(idx < 0) | (idx >= n)][0])
        raise IndexError(f"index {bad} out of range [0,{n}) for table {table_id}")
    which = np.searchsorted(pl.starts[table_id], idx, side="right") - 1
    return pl.servers[table_id][which]


def group_feature(pl: Placement, table_id: int, idx):
    """One feature's indices grouped by server, order-preserving, groups by
    ascending server (routing.py:117-148). Returns list of
    (server, indices, positions)."""
    idx = np.asarray(idx, dtype=np.int64)
    srv = resolve_many(pl, table_id, idx)
    out = []
    for s in np.unique(srv):
        pos = np.nonzero(srv == s)[0]
        out.append((int(s), idx[pos].tolist(), pos.tolist()))
    return out


# ---------------------------------------------------------------- workload

class ZipfSampler:
    """Inverse-CDF Zipf over rows 0..n-1, pmf ∝ (r+1)^-alpha
    (workload.py:111-126)."""

    def __init__(self, n: int, alpha: float):
        w = np.arange(1, n + 1, dtype=np.float64) ** (-alpha)
        self.n = n
        self.pmf = w / w.sum()
        self.cdf = np.cumsum(self.pmf)

    def sample(self, rng: np.random.Generator, count: int) -> np.ndarray:
        return np.searchsorted(self.cdf, rng.random(count), side="right")


# ---------------------------------------------------------------- dedup

KEY_ROW_BITS = 40


def make_keys(tables, rows) -> np.ndarray:
    """u64 key = table << 40 | row."""
    return (np.asarray(tables, dtype=np.uint64) << np.uint64(KEY_ROW_BITS)) | np.asarray(rows, dtype=np.uint64)


def dedup_keys(keys):
    """np.unique with inverse and multiplicity (SURVEY §8(c) parity contract)."""
    u, inv, cnt = np.unique(np.asarray(keys, dtype=np.uint64), return_inverse=True, return_counts=True)
    return u, inv.reshape(-1), cnt


# ---------------------------------------------------------------- cache

class MemoryModelO:
    """cache.py:37-75."""

    def __init__(self, cap, fixed, per_sample):
        self.cap, self.fixed, self.per = cap, fixed, per_sample

    def target(self, b):
        need = self.fixed + b * self.per
        if need > self.cap:
            raise OverflowError("capacity")
        return self.cap - need


class LoadTrackerO:
    """cache.py:78-111 (windowed mean / max against watermarks)."""

    def __init__(self, window=16, high=512, low=128, stat="mean"):
        self.win, self.w, self.high, self.low, self.stat = [], window, high, low, stat

    def value(self):
        if not self.win:
            return 0.0
        return sum(self.win) / len(self.win) if self.stat == "mean" else float(max(self.win))

    def record(self, b):
        self.win.append(b)
        if len(self.win) > self.w:
            self.win.pop(0)
        v = self.value()
        return "high" if v >= self.high else ("low" if v <= self.low else "normal")


class CachePolicyO:
    """cache.py:355-378."""

    def __init__(self, model: MemoryModelO, hyst=0.05):
        self.m, self.h = model, hyst

    def propose(self, cur, level, wb):
        b = max(1, int(round(wb)))
        try:
            tgt = self.m.target(b)
        except OverflowError:
            tgt = 0
        p = min(cur, tgt) if level == "high" else (max(cur, tgt) if level == "low" else tgt)
        return cur if abs(p - cur) < self.h * self.m.cap else p


class CacheOracle:
    """Restatement of AdaptiveCache + FrequencySketch (cache.py:114-352).

    Entries live in an insertion-ordered dict in LRU order, like the
    reference's OrderedDict: hits move to the end (cache.py:199-201),
    inserts append (cache.py:262-263), eviction pops the front. Row keys are
    (table, row) tuples; pooled-result keys (cache.py:204-223) are
    ("pooled", table, op, tuple(sorted(indices))). entry = [last_tick, size,
    hits, vector-or-None]."""

    def __init__(self, budget_bytes: int, admission="sketch", decay=0.5, prune=0.25, pooled=False):
        self.budget = int(budget_bytes)
        self.admission = admission
        self.decay, self.prune = decay, prune
        self.pooled = pooled
        self.used = 0
        self.tick = 0
        self.hits = 0
        self.misses = 0
        self.entries: OrderedDict = OrderedDict()
        self.sketch: dict = {}
        self.pending: list = []     # (key, size)
        self.evictions: list = []

    def _victim(self):
        return next(iter(self.entries))

    def lru_keys(self):
        return list(self.entries)

    # -- probe (cache.py:189-202)
    def get(self, key) -> bool:
        self.tick += 1
        e = self.entries.get(key)
        if e is None:
            self.misses += 1
            self.sketch[key] = self.sketch.get(key, 0.0) + 1.0
            return False
        self.hits += 1
        e[2] += 1
        e[0] = self.tick
        self.entries.move_to_end(key)
        return True

    # -- pooled-result keyspace (cache.py:204-223)
    def pooled_get(self, key):
        if not self.pooled:
            return None
        self.tick += 1
        e = self.entries.get(key)
        if e is None:
            return None
        e[2] += 1
        e[0] = self.tick
        self.entries.move_to_end(key)
        return e[3]

    def pooled_put(self, key, vector) -> None:
        if not self.pooled:
            return
        self._insert(key, int(np.asarray(vector).size) * 4, vector)

    # -- admission (cache.py:237-280)
    def offer(self, key, size) -> bool:
        if key in self.entries:
            return True
        if size > self.budget:
            return False
        if self.admission == "sketch" and self.used + size > self.budget:
            v = self._victim()
            if self.sketch.get(key, 0.0) < self.sketch.get(v, 0.0):
                return False
        return self._insert(key, size)

    def _insert(self, key, size, vector=None) -> bool:
        """cache.py:256-268. No presence check: re-inserting a resident key
        keeps its position and adds its size again (only pooled_put can)."""
        if size > self.budget:
            return False
        while self.used + size > self.budget:
            self._evict_one()       # KeyError on an empty dict, like the reference
        self.tick += 1
        self.entries[key] = [self.tick, size, 0, vector]
        self.used += size
        if self.used > self.budget:
            raise AssertionError(f"cache used {self.used} exceeds budget {self.budget}")
        return True

    def _evict_one(self):
        k, e = self.entries.popitem(last=False)
        self.used -= e[1]
        self.evictions.append(k)
        return k

    # -- resize / staging (cache.py:290-352)
    def resize(self, new_budget, row_bytes_of=None, fetch=False):
        grow = new_budget > self.budget
        self.budget = int(new_budget)
        ev = []
        while self.used > self.budget:
            ev.append(self._evict_one())
        staged = []
        if grow and fetch:
            staged = self.stage(row_bytes_of, None)
        return ev, staged

    def hottest(self, n):
        return [k for k, _ in sorted(self.sketch.items(), key=lambda kv: (-kv[1], kv[0]))[:n]]

    def stage(self, row_bytes_of, limit):
        staged = []
        room = self.budget - self.used
        if room <= 0 or not self.sketch:
            return staged
        pend = {k for k, _ in self.pending}
        for key in self.hottest(limit if limit is not None else len(self.sketch)):
            if not (isinstance(key, tuple) and len(key) == 2):
                continue
            if key in self.entries or key in pend:
                continue
            size = row_bytes_of(key[0])
            if size > room:
                continue
            self.pending.append((key, size))
            staged.append(key)
            room -= size
            if limit is not None and len(staged) >= limit:
                break
        return staged

    def apply_pending(self) -> int:
        n = 0
        for key, size in self.pending:
            if key not in self.entries and self._insert(key, size):
                n += 1
        self.pending.clear()
        return n

    def age(self):
        dead = []
        for k in self.sketch:
            self.sketch[k] *= self.decay
            if self.sketch[k] < self.prune:
                dead.append(k)
        for k in dead:
            del self.sketch[k]


# ---------------------------------------------------------------- batches

@dataclass
class BagBatch:
    """A batch as CSR bags.

    bag b has table bag_table[b], op bag_op[b] ("sum"/"mean"), indices
    indices[offsets[b]:offsets[b+1]], and belongs to (bag_lookup[b],
    bag_fpos[b]) of the reference Batch (requests.py:10-46). Bags may be in
    any order; sample-major order is (lookup, fpos)."""
    offsets: np.ndarray
    indices: np.ndarray
    bag_table: np.ndarray
    bag_op: list
    bag_lookup: np.ndarray
    bag_fpos: np.ndarray
    n_lookups: int
    batch_id: int = 0

    @property
    def n_bags(self):
        return len(self.bag_table)

    def sm_order(self):
        return np.lexsort((self.bag_fpos, self.bag_lookup))

    def bag_indices(self, b):
        return self.indices[self.offsets[b]:self.offsets[b + 1]]


def bag_batch_from_lists(lookups, batch_id=0) -> BagBatch:
    """lookups: list of list of (table, op, indices) in sample-major order."""
    offs, idx, bt, bo, bl, bf = [0], [], [], [], [], []
    for li, feats in enumerate(lookups):
        for fp, (t, op, ix) in enumerate(feats):
            idx.extend(int(i) for i in ix)
            offs.append(len(idx))
            bt.append(t)
            bo.append(op)
            bl.append(li)
            bf.append(fp)
    return BagBatch(np.array(offs, np.int64), np.array(idx, np.int64), np.array(bt, np.int64),
                    bo, np.array(bl, np.int64), np.array(bf, np.int64), len(lookups), batch_id)


def flat_pool_batch(seed, dims: dict, bb: BagBatch, chunk_rows=1 << 20) -> dict:
    """Flat pooled f32 vector per bag: f64 sequential sum in index order, Mean
    divides once (ranker.py:458-465 + pooling.py:74-85), vectorised across
    bags of one table. Returns {bag: vector}."""
    out = {}
    for t in np.unique(bb.bag_table):
        bags = np.nonzero(bb.bag_table == t)[0]
        D = dims[int(t)]
        # process bags in chunks bounded by total rows
        i = 0
        while i < len(bags):
            j, rows = i, 0
            while j < len(bags) and (rows == 0 or rows + bb.offsets[bags[j] + 1] - bb.offsets[bags[j]] <= chunk_rows):
                rows += bb.offsets[bags[j] + 1] - bb.offsets[bags[j]]
                j += 1
            cb = bags[i:j]
            lens = bb.offsets[cb + 1] - bb.offsets[cb]
            allidx = np.concatenate([bb.bag_indices(b) for b in cb])
            vals = rows_of(seed, int(t), D, allidx)
            starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
            acc = np.zeros((len(cb), D), np.float64)
            for k in range(int(lens.max()) if len(lens) else 0):
                m = lens > k
                acc[m] += vals[starts[m] + k]
            for n, b in enumerate(cb):
                v = acc[n]
                if bb.bag_op[b] == "mean" and lens[n]:  # empty bags stay 0 (the reference rejects them)
                    v = v / lens[n]
                out[int(b)] = v.astype(np.float32)
            i = j
    return out


class PipelineOracle:
    """Canonical-order restatement of Ranker's per-batch pipeline
    (ranker.py:218-442) on a CSR batch:

      validate -> apply_pending -> admission check -> probe every occurrence
      in (lookup, feature, position) order -> group misses by server and plan
      -> hierarchical combine -> offer raw-fetched misses in first raw
      occurrence (lookup, feature, position) order -> maintenance
      (record -> propose -> resize(fetch) -> stage(admit_per_batch) -> age).

    With one server this order is exactly Ranker's (validated against the
    reference on 1-server/1-connection topologies in tests/golden)."""

    def __init__(self, seed, dims: dict, placement: Placement, threshold=2,
                 cache: CacheOracle | None = None, policy: CachePolicyO | None = None,
                 tracker: LoadTrackerO | None = None, adaptive=True, admit_per_batch=64):
        self.seed, self.dims, self.pl = seed, dims, placement
        self.threshold = threshold
        self.cache, self.policy, self.tracker = cache, policy, tracker
        self.adaptive, self.admit = adaptive, admit_per_batch
        self.metrics = []

    def row(self, t, r):
        return rows_of(self.seed, t, self.dims[t], [r])[0]

    def run(self, bb: BagBatch):
        c = self.cache
        for b in range(bb.n_bags):
            t = int(bb.bag_table[b])
            ix = bb.bag_indices(b)
            n = self.pl.num_rows[t]
            if ix.size and (ix.min() < 0 or ix.max() >= n):
                bad = int(ix[(ix < 0) | (ix >= n)][0])
                raise IndexError(f"batch {bb.batch_id}, lookup {int(bb.bag_lookup[b])}: index {bad} "
                                 f"out of range [0,{n}) for table {t}")
        if c is not None:
            c.apply_pending()
        if c is not None and self.policy is not None:
            m = self.policy.m
            need = m.fixed + bb.n_lookups * m.per
            if need > m.cap:
                raise OverflowError("nn capacity")
            if need + c.budget > m.cap:
                if not self.adaptive:
                    raise OverflowError("fixed cache")
                c.resize(m.target(bb.n_lookups))
        order = bb.sm_order()
        hitmask = {}
        pooled_hit = {}
        hits = misses = 0
        for b in order:
            t = int(bb.bag_table[b])
            hm = np.zeros(bb.offsets[b + 1] - bb.offsets[b], bool)
            if c is not None and c.pooled:  # ranker.py:238-245: pooled probe first
                v = c.pooled_get(("pooled", t, bb.bag_op[b], tuple(sorted(int(i) for i in bb.bag_indices(b)))))
                if v is not None:
                    pooled_hit[int(b)] = v
                    hitmask[int(b)] = np.ones_like(hm)
                    hits += hm.size
                    continue
            if c is not None:
                for k, r in enumerate(bb.bag_indices(b)):
                    hm[k] = c.get((t, int(r)))
            hitmask[int(b)] = hm
            if c is not None:  # ranker.py:241-242: no cache -> no hit/miss accounting
                hits += int(hm.sum())
                misses += int((~hm).sum())
        counters = {}
        vectors = {}
        offers = {}
        pd_groups = pd_rows = raw_rows = 0
        for b in order:
            b = int(b)
            t = int(bb.bag_table[b])
            ix = bb.bag_indices(b)
            hm = hitmask[b]
            if b in pooled_hit:  # ranker.py:403-404
                vectors[b] = pooled_hit[b]
                counters[b] = (int(hm.size), 0, 0, 0)
                continue
            miss_pos = np.nonzero(~hm)[0]
            partials, raw = [], {}
            for p in np.nonzero(hm)[0]:
                raw[int(p)] = self.row(t, int(ix[p]))
            cg = [0, 0, 0, 0]  # hits, pushdown groups, pushdown rows, raw rows
            cg[0] = int(hm.sum())
            if miss_pos.size:
                groups = group_feature(self.pl, t, ix[miss_pos])
                modes = plan_modes({g[0]: len(g[1]) for g in groups}, self.threshold)
                for srv, gidx, gpos in groups:
                    rows = rows_of(self.seed, t, self.dims[t], gidx)
                    if modes[srv] == "pushdown":
                        partials.append((seq_sum_f64(rows).astype(np.float32), len(gidx), srv))
                        cg[1] += 1
                        cg[2] += len(gidx)
                    else:
                        for q, r in zip(gpos, rows):
                            raw[int(miss_pos[q])] = r
                        cg[3] += len(gidx)
            for p in sorted(raw):
                if not hm[p]:
                    offers.setdefault((t, int(ix[p])), None)
            vectors[b] = combine_partials(partials, [raw[p] for p in sorted(raw)], bb.bag_op[b])
            if c is not None and c.pooled:  # ranker.py:412-414
                c.pooled_put(("pooled", t, bb.bag_op[b], tuple(sorted(int(i) for i in ix))), vectors[b])
            counters[b] = tuple(cg)
            pd_groups += cg[1]
            pd_rows += cg[2]
            raw_rows += cg[3]
        if c is not None:
            for key in offers:
                c.offer(key, self.dims[key[0]] * 4)
        level = None
        if c is not None and self.tracker is not None and self.policy is not None:
            level = self.tracker.record(bb.n_lookups)
            if self.adaptive:
                rb = lambda t: self.dims[t] * 4
                prop = self.policy.propose(c.budget, level, self.tracker.value())
                if prop != c.budget:
                    c.resize(prop, rb, fetch=True)
                if self.admit > 0:
                    c.stage(rb, self.admit)
                c.age()
        self.metrics.append(dict(batch_id=bb.batch_id, size=bb.n_lookups, hits=hits, misses=misses,
                                 pushdown_groups=pd_groups, pushdown_rows=pd_rows, raw_rows=raw_rows,
                                 load_level=level, offers=list(offers), pooled_hits=sorted(pooled_hit)))
        return vectors, counters, hitmask
