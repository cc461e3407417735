"""Adaptive hot-row cache (mirror of embserve/cache.py).

MemoryModel / LoadTracker / CachePolicy are host-side scalar control logic
with the reference's semantics (cache.py:37-111, 355-378). AdaptiveCache and
FrequencySketch are GPU-resident: a libflexemb `fx_cache` handle holds the
hash index, slot rows, LRU ticks and the exact decayed-frequency sketch in
HBM, and K3/K6 kernels implement get/offer/resize/stage/apply/age with the
reference's ordering (see csrc/fx_cache.cu). Keys are (table, row) tuples on
the Python side and u64 `table << 40 | row` on the device.
"""

from __future__ import annotations

import ctypes
import weakref
from collections import deque
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _lib
from .errors import CapacityError, ConfigError, InvariantError

ROW_BITS = 40


class LoadLevel(Enum):
    HIGH = "high"
    NORMAL = "normal"
    LOW = "low"


@dataclass(frozen=True)
class MemoryModel:
    """NN memory is affine in batch size; the cache gets the rest (cache.py:37-50)."""

    gpu_capacity_bytes: int
    nn_fixed_bytes: int
    nn_per_sample_bytes: int

    def __post_init__(self):
        if min(self.gpu_capacity_bytes, self.nn_fixed_bytes, self.nn_per_sample_bytes) < 0:
            raise ConfigError("memory model coefficients must be >= 0")
        if self.nn_fixed_bytes > self.gpu_capacity_bytes:
            raise ConfigError("nn_fixed_bytes exceeds gpu_capacity_bytes")

    def nn_bytes(self, batch_size: int) -> int:
        return self.nn_fixed_bytes + batch_size * self.nn_per_sample_bytes


def target_cache_bytes(model: MemoryModel, batch_size: int) -> int:
    need = model.nn_bytes(batch_size)
    if need > model.gpu_capacity_bytes:
        raise CapacityError(f"batch {batch_size} needs {need} NN bytes, capacity is {model.gpu_capacity_bytes}")
    return model.gpu_capacity_bytes - need


def max_batch_for_cache(model: MemoryModel, cache_bytes: int) -> int:
    if cache_bytes + model.nn_fixed_bytes > model.gpu_capacity_bytes:
        raise CapacityError(f"cache {cache_bytes} plus fixed NN {model.nn_fixed_bytes} exceeds "
                            f"capacity {model.gpu_capacity_bytes}")
    if model.nn_per_sample_bytes == 0:
        raise ConfigError("nn_per_sample_bytes must be > 0 to bound batch size")
    return (model.gpu_capacity_bytes - cache_bytes - model.nn_fixed_bytes) // model.nn_per_sample_bytes


class LoadTracker:
    """Windowed mean (or max) of recent batch sizes vs two watermarks (cache.py:78-111)."""

    def __init__(self, window: int = 16, high_watermark: int = 512, low_watermark: int = 128, stat: str = "mean"):
        if low_watermark >= high_watermark:
            raise ConfigError("low_watermark must be < high_watermark")
        if stat not in ("mean", "max"):
            raise ConfigError(f"unknown window stat '{stat}'")
        self.window: deque = deque(maxlen=window)
        self.high_watermark = high_watermark
        self.low_watermark = low_watermark
        self.stat = stat

    def record_batch(self, batch_size: int) -> LoadLevel:
        if batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        self.window.append(batch_size)
        return self.classify()

    def windowed_value(self) -> float:
        if not self.window:
            return 0.0
        return sum(self.window) / len(self.window) if self.stat == "mean" else float(max(self.window))

    def classify(self) -> LoadLevel:
        if not self.window:
            return LoadLevel.NORMAL
        v = self.windowed_value()
        if v >= self.high_watermark:
            return LoadLevel.HIGH
        if v <= self.low_watermark:
            return LoadLevel.LOW
        return LoadLevel.NORMAL


@dataclass
class CachePolicy:
    """Load level + windowed batch -> next budget, with hysteresis (cache.py:355-378)."""

    model: MemoryModel
    hysteresis_fraction: float = 0.05

    def propose(self, current_budget: int, level: LoadLevel, windowed_batch: float) -> int:
        batch = max(1, int(round(windowed_batch)))
        try:
            target = target_cache_bytes(self.model, batch)
        except CapacityError:
            target = 0
        if level is LoadLevel.HIGH:
            proposed = min(current_budget, target)
        elif level is LoadLevel.LOW:
            proposed = max(current_budget, target)
        else:
            proposed = target
        if abs(proposed - current_budget) < self.hysteresis_fraction * self.model.gpu_capacity_bytes:
            return current_budget
        return proposed


@dataclass
class ResizeReport:
    old_budget: int
    new_budget: int
    evicted: list = field(default_factory=list)
    admitted: list = field(default_factory=list)
    applied: bool = True


_SC = ("budget", "used", "tick", "hits", "misses", "entries", "free_top", "sketch_live", "sketch_tomb",
       "hash_tomb", "pending", "n_evlog", "n_acc", "n_ev", "n_cand", "staged", "err", "n_ov", "n_par_puts", "tiles_bulk", "tiles_chain")

POOLED_BIT = 1 << 63


def encode_key(table_id: int, index: int) -> int:
    return (int(table_id) << ROW_BITS) | int(index)


def decode_key(k: int, pooled_names: dict | None = None):
    """Row key -> (table, row); pooled fingerprint -> the reference's
    ("pooled", table, op, sorted indices) key when known, else ("pooled", A)."""
    k = int(k) & ((1 << 64) - 1)
    if k & POOLED_BIT:
        if pooled_names is not None and k in pooled_names:
            return pooled_names[k]
        return ("pooled", k)
    return (k >> ROW_BITS, k & ((1 << ROW_BITS) - 1))


def bag_fingerprints(bag_table: torch.Tensor, bag_op: torch.Tensor, indices: torch.Tensor, offsets: torch.Tensor):
    """Pooled-result keys (A, B) of every CSR bag (fx_bag_fingerprint)."""
    n = int(offsets.numel()) - 1
    dev = offsets.device
    ka = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    kb = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    if n > 0:
        idx = indices if indices.numel() else torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(_lib.lib.fx_bag_fingerprint(bag_table.data_ptr(), bag_op.data_ptr(), idx.data_ptr(),
                                               _lib.idx_type_of(idx), offsets.data_ptr(), n, ka.data_ptr(),
                                               kb.data_ptr(), _lib.stream_ptr()), "bag fingerprint")
    return ka[:n], kb[:n]


def _u64(keys) -> torch.Tensor:
    arr = np.asarray([k if k < (1 << 63) else k - (1 << 64) for k in keys], dtype=np.int64)
    return torch.from_numpy(arr)


def _sig():
    L = _lib.lib
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sigs = {
        "fx_cache_create": [ctypes.POINTER(ctypes.c_void_p), I64, I32, I32, D, D, I64, I64, I32],
        "fx_cache_destroy": [P],
        "fx_cache_set_tables": [P, P, I32, P, I32],
        "fx_cache_scalars": [P, P, P],
        "fx_cache_reserve_sketch": [P, I64, P],
        "fx_cache_reserve_slots": [P, I64, P],
        "fx_cache_probe": [P, P, P, P, P, I64, I64, P, P],
        "fx_cache_offer": [P, P, I64, P, P, P, P],
        "fx_cache_set_budget": [P, I64, P],
        "fx_cache_stage": [P, I64, ctypes.POINTER(I64), P],
        "fx_cache_apply_pending": [P, ctypes.POINTER(I64), P],
        "fx_cache_age": [P, P],
        "fx_cache_lookup": [P, P, I64, P, I32, P, P],
        "fx_cache_sketch_estimate": [P, P, I64, P, P],
        "fx_cache_sketch_bump": [P, P, P, I64, P],
        "fx_cache_sketch_ranked": [P, P, P, I64, ctypes.POINTER(I64), P],
        "fx_cache_lru": [P, P, P, P, I64, ctypes.POINTER(I64), P],
        "fx_cache_eviction_log": [P, P, I64, ctypes.POINTER(I64), P],
        "fx_cache_pending": [P, P, I64, ctypes.POINTER(I64), P],
        "fx_cache_last_evicted": [P, P, I64, ctypes.POINTER(I64), P],
        "fx_cache_set_pending_rows": [P, P, I64],
        "fx_cache_set_parallel": [P, I32],
        "fx_cache_advance_tick": [P, I64, P],
        "fx_cache_rows": [P, ctypes.POINTER(P), ctypes.POINTER(I64)],
        "fx_cache_pooled_find": [P, P, P, I64, P, P],
        "fx_cache_pooled_touch": [P, P, P, I64, P],
        "fx_cache_read_slots": [P, P, I64, P, I32, P, P],
        "fx_cache_pooled_put": [P, P, P, I64, P, I32, P, P],
        "fx_cache_scalars_device": [P],
        "fx_cache_capacity": [P, P],
        "fx_cache_queue_valid": [P],
    }
    for n, a in sigs.items():
        f = getattr(L, n)
        f.argtypes = a
        f.restype = ctypes.c_void_p if n == "fx_cache_scalars_device" else ctypes.c_int
    return L


class FxTableDir(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("ld", ctypes.c_int64), ("table", ctypes.c_int32), ("dim", ctypes.c_int32)]


class FrequencySketch:
    """View of the device sketch (cache.py:114-144): exact decayed counts."""

    def __init__(self, cache: "AdaptiveCache", decay: float, prune_below: float = 0.25):
        # a weak back-reference: a cache <-> sketch cycle would keep the
        # device buffers alive after `del cache` until the next GC pass
        self._c = weakref.proxy(cache)
        self.decay = decay
        self.prune_below = prune_below

    def bump(self, key, weight: float = 1.0) -> None:
        c = self._c
        c._reserve_sketch(1)
        k = _u64([encode_key(*key)]).to(c.device)
        w = torch.tensor([float(weight)], dtype=torch.float64, device=c.device)
        _lib.check(c._L.fx_cache_sketch_bump(c._h, k.data_ptr(), w.data_ptr(), 1, _lib.stream_ptr()), "sketch bump")

    def estimate(self, key) -> float:
        c = self._c
        k = _u64([encode_key(*key)]).to(c.device)
        out = torch.empty(1, dtype=torch.float64, device=c.device)
        _lib.check(c._L.fx_cache_sketch_estimate(c._h, k.data_ptr(), 1, out.data_ptr(), _lib.stream_ptr()),
                   "sketch estimate")
        return float(out.item())

    def age(self) -> None:
        _lib.check(self._c._L.fx_cache_age(self._c._h, _lib.stream_ptr()), "sketch age")

    def ranked(self):
        """[(key, count)] sorted by (-count, key) — FrequencySketch.hottest order."""
        c = self._c
        n_live = c._scalars()["sketch_live"]
        cap = max(1, n_live)
        keys = torch.empty(cap, dtype=torch.int64, device=c.device)
        vals = torch.empty(cap, dtype=torch.float64, device=c.device)
        n = ctypes.c_int64(0)
        _lib.check(c._L.fx_cache_sketch_ranked(c._h, keys.data_ptr(), vals.data_ptr(), cap, ctypes.byref(n),
                                               _lib.stream_ptr()), "sketch ranked")
        k = keys[:n.value].cpu().numpy().view(np.uint64)
        v = vals[:n.value].cpu().numpy()
        return [(decode_key(int(a)), float(b)) for a, b in zip(k, v)]

    def ranked_arrays(self):
        """[sync] (u64 keys, f64 counts) numpy arrays in (-count, key) order."""
        c = self._c
        n_live = c._scalars()["sketch_live"]
        cap = max(1, n_live)
        keys = torch.empty(cap, dtype=torch.int64, device=c.device)
        vals = torch.empty(cap, dtype=torch.float64, device=c.device)
        n = ctypes.c_int64(0)
        _lib.check(c._L.fx_cache_sketch_ranked(c._h, keys.data_ptr(), vals.data_ptr(), cap, ctypes.byref(n),
                                               _lib.stream_ptr()), "sketch ranked")
        return keys[:n.value].cpu().numpy().view(np.uint64), vals[:n.value].cpu().numpy()

    def hottest(self, n: int, exclude=()) -> list:
        skip = set(exclude)
        return [k for k, _ in self.ranked() if k not in skip][:n]

    @property
    def _counts(self) -> dict:
        return dict(self.ranked())

    def __len__(self):
        return self._c._scalars()["sketch_live"]


class AdaptiveCache:
    """GPU-resident byte-budgeted LRU cache with decayed-frequency admission
    (cache.py:164-352). `slot_capacity` bounds the number of resident rows
    (grown on demand when the budget allows more); `max_dim` bounds row width."""

    def __init__(self, budget_bytes: int, admission: str = "sketch", sketch_decay: float = 0.5,
                 pooled_results: bool = False, record_evictions: bool = False, *, max_dim: int = 256,
                 slot_capacity: int | None = None, sketch_capacity: int = 4096, device=None):
        if admission not in ("sketch", "always"):
            raise ConfigError(f"unknown admission policy '{admission}'")
        self._L = _sig()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.admission = admission
        self.pooled_results_enabled = bool(pooled_results)
        self._pooled_names: dict = {}   # fingerprint A -> reference key (API puts)
        self.record_evictions = record_evictions
        self.max_dim = max_dim
        self._row_bytes: dict = {}      # table -> row bytes (device tbytes)
        self._dir: list = []            # FxTableDir entries
        self._pending_src: dict = {}    # key -> device vector from a Python fetcher
        self._keepalive: list = []
        if slot_capacity is None:
            slot_capacity = max(64, min(int(budget_bytes) // 4 + 1, 1 << 16))
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._L.fx_cache_create(ctypes.byref(h), int(slot_capacity), int(max_dim),
                                               0 if admission == "sketch" else 1, float(sketch_decay), 0.25,
                                               int(budget_bytes), int(sketch_capacity),
                                               1 if record_evictions else 0), "cache create")
        self._h = h
        self._slots = int(slot_capacity)
        self._budget = int(budget_bytes)   # host mirror: the budget only changes through resize()
        self.sketch = FrequencySketch(self, sketch_decay)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self._L.fx_cache_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # -- device plumbing --------------------------------------------------------

    def _scalars(self) -> dict:
        out = (ctypes.c_int64 * len(_SC))()
        _lib.check(self._L.fx_cache_scalars(self._h, out, _lib.stream_ptr()), "cache scalars")
        return dict(zip(_SC, list(out)))

    def _queue_valid_host(self) -> bool:
        """False after a staged-pipeline call moved entries (the fused step
        then rebuilds its LRU queue on the host before launching — not
        possible inside a captured graph)."""
        return bool(self._L.fx_cache_queue_valid(self._h))

    def capacity(self) -> dict:
        out = (ctypes.c_int64 * 3)()
        _lib.check(self._L.fx_cache_capacity(self._h, out), "cache capacity")
        return dict(slots=out[0], index=out[1], sketch=out[2])

    def scalars_tensor(self) -> torch.Tensor:
        """Zero-copy int64 view of the device scalars (_SC order), for async snapshots."""
        from .step import _dev_view
        return _dev_view(self._L.fx_cache_scalars_device(self._h), len(_SC), self.device)

    def _reserve_sketch(self, n_new: int):
        _lib.check(self._L.fx_cache_reserve_sketch(self._h, int(n_new), _lib.stream_ptr()), "reserve sketch")

    def _reserve_slots_for(self, budget: int, extra_size: int | None = None):
        sizes = [b for b in self._row_bytes.values() if b > 0] + ([int(extra_size)] if extra_size else [])
        sizes = sizes or [4]
        need = budget // min(sizes) + 1
        if need > self._slots:
            new = max(need, 2 * self._slots)
            _lib.check(self._L.fx_cache_reserve_slots(self._h, int(new), _lib.stream_ptr()), "reserve slots")
            self._slots = new

    def _upload_tables(self):
        n_t = (max(self._row_bytes) + 1) if self._row_bytes else 0
        tb = (ctypes.c_int32 * max(n_t, 1))(*([-1] * max(n_t, 1)))
        for t, b in self._row_bytes.items():
            tb[t] = b
        dirs = (FxTableDir * max(len(self._dir), 1))(*self._dir)
        _lib.check(self._L.fx_cache_set_tables(self._h, dirs, len(self._dir), tb, n_t), "cache tables")

    def set_parallel_offers(self, on: bool) -> None:
        """Exact run-parallel ordered offers (uniform row size) vs the
        sequential reference loop; both give identical results."""
        _lib.check(self._L.fx_cache_set_parallel(self._h, 1 if on else 0), "set parallel")

    def set_row_bytes(self, table_id: int, nbytes: int):
        if self._row_bytes.get(table_id) != nbytes:
            if nbytes > 4 * self.max_dim:
                raise ConfigError(f"row of {nbytes} bytes exceeds the cache's max_dim {self.max_dim}")
            self._row_bytes[table_id] = int(nbytes)
            self._upload_tables()

    def bind_tables(self, deployment) -> None:
        """Register where each table's rows live on this GPU (admission fetches
        read them on the device, like Deployment.get_row, store.py:215-225)."""
        self._dir = []
        for sid, server in deployment.servers.items():
            for t in server.hosted_tables():
                for sh in server.shards(t):
                    if sh.data is None or sh.data.device != self.device:
                        continue
                    self._dir.append(FxTableDir(sh.data.data_ptr(), sh.start, sh.end, sh.data.stride(0), t,
                                                sh.data.shape[1]))
                    self._keepalive.append(sh.data)
        for t, m in deployment.metas.items():
            self._row_bytes[t] = m.row_bytes
        self._upload_tables()
        self._reserve_slots_for(self.budget_bytes)

    # -- scalar state ---------------------------------------------------------------

    @property
    def budget_bytes(self) -> int:
        return self._budget

    @property
    def used_bytes(self) -> int:
        return self._scalars()["used"]

    @property
    def tick(self) -> int:
        return self._scalars()["tick"]

    @property
    def hits(self) -> int:
        return self._scalars()["hits"]

    @property
    def misses(self) -> int:
        return self._scalars()["misses"]

    def hit_rate(self) -> float:
        s = self._scalars()
        t = s["hits"] + s["misses"]
        return s["hits"] / t if t else 0.0

    def __len__(self) -> int:
        return self._scalars()["entries"]

    def __bool__(self) -> bool:
        # the reference's `if self.cache` relies on __len__ (ranker.py:397-399)
        return len(self) > 0

    def contains(self, table_id: int, index: int) -> bool:
        return self._lookup([encode_key(table_id, index)])[0] >= 0

    def _lookup(self, keys, want_rows=False):
        k = _u64(keys).to(self.device)
        slot = torch.empty(len(keys), dtype=torch.int32, device=self.device)
        rows = torch.zeros((len(keys), self.max_dim), dtype=torch.float32, device=self.device)
        _lib.check(self._L.fx_cache_lookup(self._h, k.data_ptr(), len(keys), rows.data_ptr(), self.max_dim,
                                           slot.data_ptr(), _lib.stream_ptr()), "cache lookup")
        s = slot.cpu().numpy()
        return (s, rows) if want_rows else s

    def lru_entries(self):
        """[(key, last_tick, hits)] in LRU order (== OrderedDict order)."""
        n_e = self._scalars()["entries"]
        cap = max(1, n_e)
        keys = torch.empty(cap, dtype=torch.int64, device=self.device)
        ticks = torch.empty(cap, dtype=torch.int64, device=self.device)
        hits = torch.empty(cap, dtype=torch.int32, device=self.device)
        n = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_lru(self._h, keys.data_ptr(), ticks.data_ptr(), hits.data_ptr(), cap,
                                        ctypes.byref(n), _lib.stream_ptr()), "cache lru")
        k = keys[:n.value].cpu().numpy().view(np.uint64)
        return [(decode_key(int(a), self._pooled_names), int(t), int(h)) for a, t, h in
                zip(k, ticks[:n.value].cpu().numpy(), hits[:n.value].cpu().numpy())]

    def lru_arrays(self):
        """[sync] (u64 keys, int64 last_tick, int32 hits) numpy arrays in LRU order."""
        n_e = self._scalars()["entries"]
        cap = max(1, n_e)
        keys = torch.empty(cap, dtype=torch.int64, device=self.device)
        ticks = torch.empty(cap, dtype=torch.int64, device=self.device)
        hits = torch.empty(cap, dtype=torch.int32, device=self.device)
        n = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_lru(self._h, keys.data_ptr(), ticks.data_ptr(), hits.data_ptr(), cap,
                                        ctypes.byref(n), _lib.stream_ptr()), "cache lru")
        k = n.value
        return keys[:k].cpu().numpy().view(np.uint64), ticks[:k].cpu().numpy(), hits[:k].cpu().numpy()

    def eviction_log_array(self):
        """[sync] the eviction log as a u64 numpy array (record_evictions=True)."""
        n_tot = self._scalars()["n_evlog"]
        cap = max(1, n_tot)
        out = torch.empty(cap, dtype=torch.int64, device=self.device)
        n = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_eviction_log(self._h, out.data_ptr(), cap, ctypes.byref(n), _lib.stream_ptr()),
                   "eviction log")
        if n.value > cap:
            raise InvariantError("eviction log overflowed its device buffer")
        return out[:n.value].cpu().numpy().view(np.uint64)

    def sketch_arrays(self):
        """[sync] (u64 keys sorted ascending, f64 counts) of the live sketch."""
        ranked = self.sketch.ranked_arrays()
        k, v = ranked
        o = np.argsort(k, kind="stable")
        return k[o], v[o]

    def lru_keys(self) -> list:
        return [e[0] for e in self.lru_entries()]

    @property
    def eviction_log(self):
        if not self.record_evictions:
            return None
        n_tot = self._scalars()["n_evlog"]
        cap = max(1, n_tot)
        out = torch.empty(cap, dtype=torch.int64, device=self.device)
        n = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_eviction_log(self._h, out.data_ptr(), cap, ctypes.byref(n), _lib.stream_ptr()),
                   "eviction log")
        if n.value > cap:
            raise InvariantError("eviction log overflowed its device buffer")
        return [decode_key(int(a), self._pooled_names) for a in out[:n.value].cpu().numpy().view(np.uint64)]

    def _last_evicted(self):
        s = self._scalars()
        cap = max(1, s["n_ev"])
        out = torch.empty(cap, dtype=torch.int64, device=self.device)
        n = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_last_evicted(self._h, out.data_ptr(), cap, ctypes.byref(n), _lib.stream_ptr()),
                   "last evicted")
        return [decode_key(int(a), self._pooled_names) for a in out[:n.value].cpu().numpy().view(np.uint64)]

    # -- batched device API (used by the engine) ------------------------------------------

    def probe_unique(self, uniq: torch.Tensor, mult: torch.Tensor, last_ord: torch.Tensor, n_uniq_dev, nnz: int,
                     slot_out: torch.Tensor | None = None, n_uniq_host: int = 0):
        """K3 over a batch's unique keys (first-occurrence order from fx_dedup).
        `nnz` is the tick advance (every probe of the batch); the sketch can
        gain at most one new key per unique key."""
        self._reserve_sketch(n_uniq_host if (n_uniq_dev is None and n_uniq_host) else nnz)
        _lib.check(self._L.fx_cache_probe(self._h, uniq.data_ptr(), mult.data_ptr(), last_ord.data_ptr(),
                                          _lib.ptr(n_uniq_dev), int(n_uniq_host), int(nnz), _lib.ptr(slot_out),
                                          _lib.stream_ptr()), "cache probe")

    def offer_keys(self, keys: torch.Tensor, n: int, src_rows: torch.Tensor | None = None,
                   accepted: torch.Tensor | None = None):
        """Ordered offers of device keys (rows from the table directory or
        src_rows pointers)."""
        _lib.check(self._L.fx_cache_offer(self._h, keys.data_ptr(), int(n), None, _lib.ptr(src_rows),
                                          _lib.ptr(accepted), _lib.stream_ptr()), "cache offer")

    # -- reference API -------------------------------------------------------------------

    def get(self, table_id: int, index: int):
        """Row probe: hit refreshes recency, miss feeds the sketch (cache.py:189-202)."""
        key = encode_key(table_id, index)
        dev = self.device
        u = _u64([key]).to(dev)
        mult = torch.ones(1, dtype=torch.int32, device=dev)
        lo = torch.zeros(1, dtype=torch.int64, device=dev)
        slot = torch.empty(1, dtype=torch.int32, device=dev)
        self.probe_unique(u, mult, lo, None, 1, slot, n_uniq_host=1)
        s = int(slot.item())
        if s < 0:
            return None
        _, rows = self._lookup([key], want_rows=True)
        dim = self._row_bytes.get(table_id, 4 * self.max_dim) // 4
        return rows[0, :dim].cpu().numpy()

    # -- pooled-result keyspace (cache.py:204-223) --------------------------------------

    def check_state(self) -> None:
        """[sync] Raise what the reference raises when a cache operation hit
        one of its failure paths (recorded device-side in scalars.err)."""
        err = self._scalars()["err"]
        if err == 1:
            raise KeyError("popitem(): dictionary is empty (cache.py:270: nothing left to evict; "
                           "leaked pooled bytes exceed the budget)")
        if err == 2:
            raise InvariantError("pooled-result key fingerprint collision (different index multisets share A)")

    def _pooled_key(self, table_id: int, op, indices):
        from .pooling import op_code
        dev = self.device
        idx = torch.as_tensor(np.asarray(list(indices), dtype=np.int64)).to(dev)
        offs = torch.tensor([0, idx.numel()], dtype=torch.int64, device=dev)
        bt = torch.tensor([int(table_id)], dtype=torch.int32, device=dev)
        bo = torch.tensor([op_code(op)], dtype=torch.int32, device=dev)
        ka, kb = bag_fingerprints(bt, bo, idx, offs)
        opv = op.value if hasattr(op, "value") else str(op)
        name = ("pooled", int(table_id), opv, tuple(sorted(int(i) for i in indices)))
        return ka, kb, name

    def pooled_find(self, key_a: torch.Tensor, key_b: torch.Tensor, slot_out: torch.Tensor) -> None:
        n = int(key_a.numel())
        if n:
            _lib.check(self._L.fx_cache_pooled_find(self._h, key_a.data_ptr(), key_b.data_ptr(), n,
                                                    slot_out.data_ptr(), _lib.stream_ptr()), "pooled find")

    def pooled_touch(self, slot: torch.Tensor, pos: torch.Tensor) -> None:
        n = int(slot.numel())
        if n:
            _lib.check(self._L.fx_cache_pooled_touch(self._h, slot.data_ptr(), pos.data_ptr(), n,
                                                     _lib.stream_ptr()), "pooled touch")

    def rows_base(self):
        """(device pointer, row stride in floats) of the slot row storage."""
        p, ld = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(self._L.fx_cache_rows(self._h, ctypes.byref(p), ctypes.byref(ld)), "cache rows")
        return int(p.value or 0), int(ld.value)

    def bind_dir(self, entries) -> None:
        """Register row locations [(base_ptr, row_begin, row_end, ld, table, dim)]
        — e.g. IPC-mapped shards of peer GPUs, read over NVLink by admissions."""
        self._dir = [FxTableDir(*e) for e in entries]
        for e in entries:
            self._row_bytes[int(e[4])] = int(e[5]) * 4
        self._upload_tables()
        self._reserve_slots_for(self.budget_bytes)

    def advance_tick(self, n: int) -> None:
        if n:
            _lib.check(self._L.fx_cache_advance_tick(self._h, int(n), _lib.stream_ptr()), "advance tick")

    def read_slots(self, slot: torch.Tensor, out: torch.Tensor, sizes: torch.Tensor | None = None) -> None:
        n = int(slot.numel())
        if n:
            _lib.check(self._L.fx_cache_read_slots(self._h, slot.data_ptr(), n, out.data_ptr(), out.stride(0),
                                                   _lib.ptr(sizes), _lib.stream_ptr()), "read slots")

    def pooled_put_many(self, key_a: torch.Tensor, key_b: torch.Tensor, rows: torch.Tensor,
                        nbytes: int, sel: torch.Tensor | None = None) -> None:
        """Ordered pooled_put of rows[i] (or rows[sel[i]]) under keys (A, B)[i]."""
        n = int(key_a.numel())
        if n == 0:
            return
        self._reserve_slots_for(self.budget_bytes, int(nbytes))
        base = rows.data_ptr()
        stride = rows.stride(0) * rows.element_size()
        rid = sel if sel is not None else torch.arange(n, device=self.device)
        ptrs = (rid.to(torch.int64) * stride + base).contiguous()
        _lib.check(self._L.fx_cache_pooled_put(self._h, key_a.data_ptr(), key_b.data_ptr(), n, None, int(nbytes),
                                               ptrs.data_ptr(), _lib.stream_ptr()), "pooled put")

    def pooled_get(self, table_id: int, op, indices):
        """Pooled-result probe (cache.py:204-217): disabled -> None without a
        tick; otherwise tick += 1, hit refreshes recency and returns the vector."""
        if not self.pooled_results_enabled:
            return None
        ka, kb, _ = self._pooled_key(table_id, op, indices)
        slot = torch.empty(1, dtype=torch.int32, device=self.device)
        self.pooled_find(ka, kb, slot)
        self.pooled_touch(slot, torch.zeros(1, dtype=torch.int64, device=self.device))
        self.advance_tick(1)
        self.check_state()
        if int(slot.item()) < 0:
            return None
        out = torch.zeros((1, self.max_dim), dtype=torch.float32, device=self.device)
        size = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.read_slots(slot, out, size)
        return out[0, :int(size.item()) // 4].cpu().numpy()

    def pooled_put(self, table_id: int, op, indices, vector) -> None:
        """cache.py:219-223: unconditional insert of a pooled vector."""
        if not self.pooled_results_enabled:
            return
        vec = vector if isinstance(vector, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(vector))
        vec = vec.to(device=self.device, dtype=torch.float32).reshape(1, -1).contiguous()
        ka, kb, name = self._pooled_key(table_id, op, indices)
        self._pooled_names[int(ka.item()) & ((1 << 64) - 1)] = name
        if vec.numel() > self.max_dim:
            raise ConfigError(f"pooled vector of {vec.numel()} floats exceeds the cache's max_dim {self.max_dim}")
        self.pooled_put_many(ka, kb, vec, vec.numel() * 4)
        self.check_state()

    def offer(self, table_id: int, index: int, vector) -> bool:
        """Admission attempt for a raw-fetched row (cache.py:237-254)."""
        vec = vector if isinstance(vector, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(vector))
        vec = vec.to(device=self.device, dtype=torch.float32).reshape(-1).contiguous()
        self.set_row_bytes(table_id, vec.numel() * 4)
        self._reserve_slots_for(self.budget_bytes)
        k = _u64([encode_key(table_id, index)]).to(self.device)
        src = torch.tensor([vec.data_ptr()], dtype=torch.int64, device=self.device)
        acc = torch.zeros(1, dtype=torch.uint8, device=self.device)
        self.offer_keys(k, 1, src, acc)
        return bool(acc.item())

    def evict_to_budget(self) -> list:
        _lib.check(self._L.fx_cache_set_budget(self._h, self.budget_bytes, _lib.stream_ptr()), "evict")
        return self._last_evicted()

    def resize(self, new_budget: int, fetcher, row_bytes_of=None) -> ResizeReport:
        """Shrink evicts LRU to the new budget; grow stages the hottest absent
        rows that fit (cache.py:290-309)."""
        if new_budget < 0:
            raise ConfigError("cache budget must be >= 0")
        old = self.budget_bytes
        rep = ResizeReport(old_budget=old, new_budget=int(new_budget))
        self._reserve_slots_for(int(new_budget))
        _lib.check(self._L.fx_cache_set_budget(self._h, int(new_budget), _lib.stream_ptr()), "resize")
        self._budget = int(new_budget)
        if self._scalars()["n_ev"]:
            rep.evicted = self._last_evicted()
        if new_budget > old and fetcher is not None:
            rep.admitted = self.stage_hot_admissions(fetcher, row_bytes_of)
        return rep

    def stage_hot_admissions(self, fetcher, row_bytes_of=None, limit: int | None = None) -> list:
        """Stage the hottest absent rows that fit the spare budget (cache.py:311-342)."""
        if row_bytes_of is not None:
            for t in list(self._row_bytes) or []:
                self.set_row_bytes(t, int(row_bytes_of(t)))
        # tables the device does not know a row size for (no deployment bound):
        # learn it the way the reference does — row_bytes_of(t), else the size
        # of the fetched vector (cache.py:327-336)
        keys, _ = self.sketch.ranked_arrays()
        if keys.size:
            rows_of_t = {}
            for k in keys.tolist():
                if k & POOLED_BIT:
                    continue
                rows_of_t.setdefault(k >> ROW_BITS, k & ((1 << ROW_BITS) - 1))
            for t, r in rows_of_t.items():
                if t in self._row_bytes:
                    continue
                if row_bytes_of is not None:
                    self.set_row_bytes(t, int(row_bytes_of(t)))
                elif fetcher is not None:
                    vv = fetcher(t, r)
                    if vv is not None:
                        self.set_row_bytes(t, int(np.asarray(vv).size) * int(np.asarray(vv).itemsize))
        before = self._scalars()["pending"]
        staged = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_stage(self._h, -1 if limit is None else int(limit), ctypes.byref(staged),
                                          _lib.stream_ptr()), "stage")
        if staged.value == 0:
            return []
        keys = self._pending_keys()[before:before + staged.value]
        known = {d.table for d in self._dir}
        for key in keys:
            if key[0] not in known and fetcher is not None:
                v = fetcher(key[0], key[1])
                t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(self.device)
                self._pending_src[key] = t
        return keys

    def _pending_keys(self):
        n_p = self._scalars()["pending"]
        cap = max(1, n_p)
        out = torch.empty(cap, dtype=torch.int64, device=self.device)
        n = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_pending(self._h, out.data_ptr(), cap, ctypes.byref(n), _lib.stream_ptr()),
                   "pending")
        return [decode_key(int(a)) for a in out[:n.value].cpu().numpy().view(np.uint64)]

    def apply_pending_admissions(self) -> int:
        """Install the rows staged by the last maintenance (cache.py:344-352)."""
        if self._pending_src:
            # rows fetched by a host fetcher: insert them through ordered offers
            # with "always" semantics via the pending path's row pointers
            keys = self._pending_keys()
            ptrs = [self._pending_src[k].data_ptr() if k in self._pending_src else 0 for k in keys]
            self._set_pending_rows(ptrs)
        applied = ctypes.c_int64(0)
        _lib.check(self._L.fx_cache_apply_pending(self._h, ctypes.byref(applied), _lib.stream_ptr()), "apply")
        self._pending_src.clear()
        self._pending_rows = None
        return applied.value

    def _set_pending_rows(self, ptrs):
        self._pending_rows = torch.tensor(ptrs, dtype=torch.int64, device=self.device)
        _lib.check(self._L.fx_cache_set_pending_rows(self._h, self._pending_rows.data_ptr(), len(ptrs)),
                   "pending rows")
