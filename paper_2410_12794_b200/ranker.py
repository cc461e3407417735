"""Batch pipeline (mirror of embserve/ranker.py) on one GPU.

Per batch, in the reference's canonical order (ranker.py:218-442; SURVEY
§8(c)):

  1. ingress validation + range routing of every index (K1 fx_route);
  2. cache.apply_pending_admissions, admission check (host scalars);
  3. dedup (K2 fx_dedup) and one cache probe per unique key (K3), equivalent
     to probing every occurrence in (lookup, feature, position) order;
  4. per (lookup, feature, server) miss-group sizes -> pushdown plan
     (threshold, pooling.py:88-100) -> counters;
  5. per-shard f64 partial pooling of the misses (K4, "pushdown near the
     data"), cache-hit rows as raw vectors, combined per bag in f64 and
     rounded once (K5) — within the reference tolerance of its hierarchical
     combine and bit-identical to the flat oracle in practice;
  6. offers of raw-fetched misses in first raw-occurrence order (K6);
  7. maintenance: record -> propose -> resize(fetch) -> stage(admit) -> age.

The modelled RDMA transport of the reference (VirtualTransport) is not
reproduced: the fan-out is a device-side bucketing of indices per shard
(streams + NCCL in the multi-GPU path, see sharded.py). `transport` is
accepted for signature compatibility and ignored.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import os

import numpy as np
import torch

from . import _lib
from .cache import AdaptiveCache, CachePolicy, LoadTracker, encode_key, target_cache_bytes
from .dedup import Deduper, sample_major_starts
from .errors import CapacityError, ConfigError, InvariantError, LookupValidationError
from .pooling import PoolingOp, op_code, pool_flat
from .requests import Batch, LookupRequest
from .store import Deployment, make_segments

_SEG_OUT = 5  # fx_segment.out, in int64 words
from .routing import RoutingTable


@dataclass
class RankerParams:
    pushdown_threshold: int | None = 2
    pipeline_depth: int = 1
    adaptive_cache: bool = True
    keep_results: bool = True
    admit_per_batch: int = 64


@dataclass
class LookupResult:
    vectors: list = field(default_factory=list)
    cache_hits: int = 0
    pushdown_groups: int = 0
    pushdown_rows: int = 0
    raw_rows: int = 0
    completed_at: float = 0.0

    @property
    def counters(self):
        return (self.cache_hits, self.pushdown_groups, self.raw_rows)


@dataclass
class BatchMetrics:
    batch_id: int
    size: int
    started_at: float
    latency: float
    subrequests: int
    cache_hits: int
    cache_misses: int
    pushdown_groups: int
    pushdown_rows: int
    raw_rows: int
    load_level: str | None = None
    cache_budget: int | None = None
    cache_used: int | None = None

    @property
    def hit_rate(self) -> float:
        t = self.cache_hits + self.cache_misses
        return self.cache_hits / t if t else 0.0


@dataclass
class CsrLayout:
    """A reference Batch packed table-major for the kernels."""
    indices: torch.Tensor     # int64 [nnz], table-major bag order
    offsets: torch.Tensor     # int64 [n_bags+1]
    bag_table: torch.Tensor   # int32 [n_bags]
    sm_start: torch.Tensor    # int64 [n_bags] (lookup, feature, position) ordinal of each bag's first index
    perm: np.ndarray          # table-major bag -> sample-major bag id
    segs: list                # [(table, op, bag_begin, bag_end)]
    lens_sm: np.ndarray       # bag lengths in sample-major order
    bag_lookup_sm: np.ndarray
    host_idx_sm: list         # per sample-major bag: host index list (error path)
    n_lookups: int


def pack_batch(batch: Batch, device) -> CsrLayout:
    tabs, ops, lk, idx_lists = [], [], [], []
    for li, lookup in enumerate(batch.lookups):
        for f in lookup.features:
            tabs.append(f.table_id)
            ops.append(op_code(f.op))
            lk.append(li)
            idx_lists.append(f.indices)
    tabs = np.asarray(tabs, np.int64)
    ops_a = np.asarray(ops, np.int64)
    lens = np.fromiter((len(x) for x in idx_lists), dtype=np.int64, count=len(idx_lists))
    perm = np.lexsort((ops_a, tabs))  # stable: table-major, sample-major within a table
    sm_start = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    lens_tm = lens[perm]
    offs = np.concatenate([[0], np.cumsum(lens_tm)]).astype(np.int64)
    flat = np.concatenate([np.asarray(idx_lists[b], dtype=np.int64) for b in perm]) if len(perm) else np.zeros(0, np.int64)
    segs = []
    tt, oo = tabs[perm], ops_a[perm]
    start = 0
    for i in range(1, len(perm) + 1):
        if i == len(perm) or tt[i] != tt[start] or oo[i] != oo[start]:
            segs.append((int(tt[start]), int(oo[start]), start, i))
            start = i
    dev = device
    return CsrLayout(torch.from_numpy(flat).to(dev), torch.from_numpy(offs).to(dev),
                     torch.from_numpy(tt.astype(np.int32)).to(dev), torch.from_numpy(sm_start[perm]).to(dev), perm,
                     segs, lens, np.asarray(lk, np.int64), idx_lists, len(batch.lookups))


def pack_csr(indices: torch.Tensor, offsets: torch.Tensor, feature_tables, feature_ops, batch_size: int,
             device) -> CsrLayout:
    """Table-major CSR (bag = f*B + s, the engine's layout) -> CsrLayout."""
    F, B = len(feature_tables), batch_size
    dev = torch.device(device)
    idx = indices.to(device=dev, dtype=torch.int64)
    offs = offsets.to(device=dev, dtype=torch.int64)
    lens = (offs[1:] - offs[:-1]).view(F, B)
    sm = (torch.cumsum(lens.t().reshape(-1), 0) - lens.t().reshape(-1)).view(B, F).t().reshape(-1).contiguous()
    ops = [op_code(o) for o in feature_ops]
    segs, b = [], 0
    for f in range(F):
        if segs and segs[-1][0] == feature_tables[f] and segs[-1][1] == ops[f]:
            segs[-1] = (segs[-1][0], segs[-1][1], segs[-1][2], b + B)
        else:
            segs.append((int(feature_tables[f]), ops[f], b, b + B))
        b += B
    bag_table = torch.tensor(np.repeat(np.asarray(feature_tables, np.int32), B), device=dev)
    return CsrLayout(idx, offs, bag_table, sm, _tm_to_sm(F, B), segs, None, None, None, B)


def _tm_to_sm(F, B):
    """perm[tm_bag] = sample-major bag id (s*F + f) for tm_bag = f*B + s."""
    f = np.repeat(np.arange(F), B)
    s_ = np.tile(np.arange(B), F)
    return s_ * F + f


class Ranker:
    def __init__(self, deployment: Deployment, routing: RoutingTable, transport=None,
                 params: RankerParams | None = None, cache: AdaptiveCache | None = None,
                 policy: CachePolicy | None = None, tracker: LoadTracker | None = None, device=None,
                 hits_from_cache: bool = True, fused: bool = True):
        self.deployment = deployment
        self.routing = routing
        self.transport = transport
        self.params = params or RankerParams()
        self.cache = cache
        self.policy = policy
        self.tracker = tracker
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.batch_metrics: list = []
        self.results: dict = {}
        self._last_level = None
        self._dedup = Deduper(self.device)
        self._status = _lib.Status(self.device)
        # device shard directory: global shard id -> (tensor, start, end, server)
        self._shards = []
        for spec in routing.shard_list:
            server = deployment.servers[spec.server_id]
            data = None
            for sh in server.shards(spec.table_id):
                if sh.start == spec.start:
                    data = sh.data
            if data is None:
                raise InvariantError(f"shard {spec} is not resident on this GPU (use sharded.ShardedLookup)")
            self._shards.append((data, spec.start, spec.end, spec.server_id, spec.table_id))
        self._server_ids = sorted({s[3] for s in self._shards})
        self._shard_server_dev = torch.tensor([self._server_ids.index(s[3]) for s in self._shards], dtype=torch.int64,
                                              device=self.device)
        if cache is not None:
            cache.bind_tables(deployment)
        # one shard per table: a single fused K4 launch pools whole bags (no
        # per-shard partials). Cache-hit rows are then read from the table copy,
        # which is bit-identical to the cached row; `hits_from_cache` keeps the
        # faithful path (hit rows read from the cache slots) when a cache is on.
        per_table = {}
        for spec in routing.shard_list:
            per_table[spec.table_id] = per_table.get(spec.table_id, 0) + 1
        self._single_shard = all(v == 1 for v in per_table.values())
        self._table_shard = {s[4]: s for s in self._shards} if self._single_shard else {}
        self.hits_from_cache = hits_from_cache
        self.profile = False
        self.stage_ms: dict = {}
        self._marks = []
        # fused, sync-free batch step (csrc/fx_step.cu) when the deployment is
        # in its domain: one full shard per table on this GPU, one row size,
        # row keys only; otherwise the staged pipeline below
        self._init_fast_state(bool(fused) and self._fast_domain())

    def _init_fast_state(self, fast: bool) -> None:
        self._fast = fast
        self._step = None
        self._engine = None
        self._pool_stream = None
        self._pending: list = []      # batches whose metrics are still on the device
        self._inflight: list = []     # started, not yet offered (pipeline_depth > 1)
        self._epoch_ev = None
        self._fast_layouts: dict = {}
        self._fast_segs: dict = {}
        self._views = None
        self.k4_events = None        # list -> (start, end) events around every K4 launch (bench roofline)

    def _mark(self, name):
        if self.profile:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._marks.append((name, ev))

    def _flush_marks(self):
        if not self.profile or not self._marks:
            return
        self._marks[-1][1].synchronize()
        for (n0, e0), (_, e1) in zip(self._marks[:-1], self._marks[1:]):
            self.stage_ms[n0] = self.stage_ms.get(n0, 0.0) + e0.elapsed_time(e1)
        self._marks = []

    # -- fused step ---------------------------------------------------------------

    def _fast_domain(self) -> bool:
        c = self.cache
        if c is None or c.pooled_results_enabled:
            return False
        dims = {m.dim for m in self.deployment.metas.values()}
        if len(dims) != 1 or max(dims) > c.max_dim:
            return False
        for t, m in self.deployment.metas.items():
            found = False
            for server in self.deployment.servers.values():
                for sh in server.shards(t):
                    if (sh.data is not None and sh.data.device == self.device and sh.start == 0
                            and sh.end == m.num_rows):
                        found = True
            if not found:
                return False
        return all(sp.start == 0 and sp.end == self.deployment.meta(sp.table_id).num_rows
                   for sp in self.routing.shard_list)

    def _admission_needs_resize(self, size: int) -> bool:
        """ranker.py:195-216 on host scalars: True when the check would raise
        or resize (those batches take the staged pipeline, which validates
        first and applies the resize in the reference's order)."""
        if self.cache is None or self.policy is None:
            return False
        model = self.policy.model
        need = model.nn_bytes(size)
        return need > model.gpu_capacity_bytes or need + self.cache.budget_bytes > model.gpu_capacity_bytes

    def _get_step(self, nnz: int, n_bags: int):
        from .step import BatchStep
        depth = max(1, int(self.params.pipeline_depth))
        st = self._step
        if (st is None or nnz > st.max_nnz or n_bags > st.max_bags or st.slots != self.cache._slots
                or st.n_slots != depth or self.params.admit_per_batch > st.stage_limit_cap):
            if self._inflight:
                raise ConfigError("a batch larger than the fused step's capacity arrived with batches in flight: "
                                  "call Ranker.reserve(max_nnz, max_bags) first")
            max_nnz = max(nnz, st.max_nnz if st else 0, 1)
            max_bags = max(n_bags, st.max_bags if st else 0, 1)
            if depth > 1:  # headroom: the step cannot grow while batches are in flight
                max_nnz, max_bags = max_nnz + max_nnz // 2, max_bags + max_bags // 2
            # the sketch must take a batch's new keys without rehashing into a
            # bigger table mid-stream (the step bakes its pointers)
            self.cache._reserve_sketch(2 * max_nnz)
            self._step = None
            self._step = BatchStep(self.cache, self.deployment, max_nnz, max_bags,
                                   stage_limit_cap=max(64, int(self.params.admit_per_batch)), slots=depth)
            self._step_slot = 0
        if self._pool_stream is None:
            self._pool_stream = torch.cuda.Stream(device=self.device)
            self._epoch_ev = torch.cuda.Event(enable_timing=True)
            self._epoch_ev.record()
        return self._step

    def reserve(self, max_nnz: int, max_bags: int) -> None:
        """Size the fused step for batches of up to `max_nnz` indices and
        `max_bags` bags (needed before streaming batches of growing size with
        pipeline_depth > 1: the step cannot grow while batches are in flight)."""
        if getattr(self, "_fast", False):
            self.sync()
            self._get_step(int(max_nnz), int(max_bags))

    def _fast_start(self, lay: CsrLayout, n_lookups: int, batch_id: int, feature_shape=None, host=None):
        """Enqueue one batch's start phase and its pooling (K4 on a side
        stream: the pooled values read only the tables). Returns the in-flight
        record; its offers/maintenance run in `_fast_finish`."""
        dev = self.device
        nnz = int(lay.indices.numel())
        n_bags = int(lay.offsets.numel()) - 1
        step = self._get_step(nnz, n_bags)
        slot = self._step_slot
        self._step_slot = (slot + 1) % step.n_slots
        cur = torch.cuda.current_stream(dev)
        D = next(iter(self.deployment.metas.values())).dim
        # outputs allocated on the caller's stream (the pooling stream only writes them)
        if feature_shape is not None:
            ft, fo, B = feature_shape
            out = torch.empty((B, len(ft) * D), dtype=torch.float32, device=dev)
        else:
            out = torch.zeros((max(n_bags, 1), D), dtype=torch.float32, device=dev)[:n_bags]
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record(cur)
        side = self._pool_stream
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            k4 = None
            if self.k4_events is not None:
                k4 = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                k4[0].record(side)
            if feature_shape is not None:
                self._pool_sample_major(lay, out, ft, fo, B)
            elif n_bags:
                self._pool_fused(lay, n_bags, out=out)
            if k4 is not None:
                k4[1].record(side)
                self.k4_events.append(k4)
        cnt = torch.empty((4, max(n_bags, 1)), dtype=torch.int32, device=dev)
        self._mark("start")
        step.start(slot, lay.bag_table, lay.indices, lay.offsets, lay.sm_start, n_bags, nnz,
                   self.params.pushdown_threshold, cnt[0], cnt[1], cnt[2], cnt[3])
        rec = dict(slot=slot, batch_id=batch_id, size=n_lookups, nnz=nnz, out=out, cnt=cnt, ev0=ev0,
                   lay=lay, host=host, feature_shape=feature_shape)
        self._inflight.append(rec)
        return rec

    def _pool_sample_major(self, lay: CsrLayout, out: torch.Tensor, ft, fo, B: int, share: bool = True) -> None:
        """One K4 launch writing out[B, F*D] sample-major (out[s, f*D:(f+1)*D]
        = bag (s, f)). The segment descriptors live on the device per batch
        shape; only their output pointers are patched per call, by a device
        op (no host->device copy, so the host never waits for the GPU).
        `share`: K4 runs beside the cache step, so it keeps at most two
        resident blocks per SM (FX_OUT_SHARE) instead of filling every SM."""
        F = len(ft)
        D = out.shape[1] // F
        seg, off = self._segs_for(ft, fo, B, D)
        seg.view(torch.int64).view(F, _lib.SEGMENT_BYTES // 8)[:, _SEG_OUT] = off + out.data_ptr()
        _lib.check(_lib.lib.fx_gather_pool(seg.data_ptr(), F, D, lay.indices.data_ptr(), _lib.idx_type_of(lay.indices),
                                           lay.offsets.data_ptr(), F * B, _lib.FX_OUT_F32 | (_lib.FX_OUT_SHARE if share else 0), None,
                                           self._status.err.data_ptr(), _lib.FX_E_LOOKUP_VALIDATION,
                                           self._status.code.data_ptr(), _lib.stream_ptr()), "gather_pool")

    def _segs_for(self, ft, fo, B: int, D: int):
        """Device segment descriptors of a batch shape (output pointers patched per call)."""
        key = (ft, fo, B)
        ent = self._fast_segs.get(key)
        F = len(ft)
        if ent is None:
            segs = []
            for f, (t, op) in enumerate(zip(ft, fo)):
                tab, start, end, _, _ = self._table_shard[t]
                segs.append(_lib.FxSegment(tab.data_ptr(), start, end, f * B, (f + 1) * B, f * D * 4, F * D,
                                           tab.stride(0), D, op_code(op)))
            seg = make_segments(segs, self.device)
            off = seg.view(torch.int64).view(F, _lib.SEGMENT_BYTES // 8)[:, _SEG_OUT].clone()
            ent = (seg, off)
            self._fast_segs[key] = ent
        return ent

    def _fast_finish(self) -> dict:
        """Offers + maintenance of the oldest in-flight batch (ranker.py:
        417-442), then an async snapshot of its metrics."""
        rec = self._inflight.pop(0)
        step, c = self._step, self.cache
        slot = rec["slot"]
        self._mark("offer")
        step.offer(slot)
        self._mark("maintain")
        level_before = (list(self.tracker.window), self._last_level) if self.tracker is not None else None
        rec["tracker_before"] = level_before
        stage_limit, age = 0, False
        if self.tracker is not None and self.policy is not None:
            level = self.tracker.record_batch(rec["size"])
            self._last_level = level.value
            if self.params.adaptive_cache:
                proposed = self.policy.propose(c.budget_bytes, level, self.tracker.windowed_value())
                if proposed != c.budget_bytes:
                    # budget change: the staged API (resize -> stage -> age) with host syncs
                    step.join()
                    self._resolve()
                    sc = step.scalars(slot)
                    if sc["err"]:
                        self._fail(rec, sc["err"], sc["err_at"])
                    rb = lambda t: self.deployment.meta(t).row_bytes
                    c.resize(proposed, fetcher=lambda t, i: self.deployment.get_row(t, i), row_bytes_of=rb)
                    if self.params.admit_per_batch > 0:
                        c.stage_hot_admissions(None, rb, limit=self.params.admit_per_batch)
                    c.sketch.age()
                    step.prepare()
                else:
                    stage_limit, age = max(0, int(self.params.admit_per_batch)), True
        if stage_limit or age:
            step.maintain(slot, stage_limit, age)
        step.join()
        self._mark("end")
        self._flush_marks()
        cur = torch.cuda.current_stream(self.device)
        cur.wait_stream(self._pool_stream)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record(cur)
        if self._views is None or self._views[0] is not step:
            self._views = (step, [step.scalars_tensor(k) for k in range(step.n_slots)], c.scalars_tensor())
        rec["snap"] = torch.cat([self._views[1][slot], self._views[2]])
        rec["ev1"] = ev1
        rec["level"] = self._last_level
        self._pending.append(rec)
        return rec

    def capture_csr(self, indices: torch.Tensor, offsets: torch.Tensor, feature_tables, feature_ops,
                    batch_size: int) -> "RankerGraph":
        """Record one whole fused Ranker batch — validation, dedup, probes,
        plan, offers, maintenance (stage + age) and the K4 pooling on its side
        stream — as ONE CUDA graph over the static device buffers `indices` /
        `offsets` (table-major CSR of fixed size). `RankerGraph.replay()`
        re-runs it on whatever the buffers hold, with the host-side policy
        bookkeeping of a normal batch; a batch whose policy would change the
        budget (or whose admission check would resize) runs eagerly instead.
        Needs the fused step and pipeline_depth 1."""
        if not getattr(self, "_fast", False) or int(self.params.pipeline_depth) != 1:
            raise ConfigError("capture_csr needs the fused step and pipeline_depth 1")
        self.sync()
        dev = self.device
        ft, fo, B = tuple(feature_tables), tuple(feature_ops), int(batch_size)
        F = len(ft)
        nnz, n_bags = int(indices.numel()), F * B
        step = self._get_step(nnz, n_bags)
        step.prepare()
        key = (ft, B)
        bt = self._fast_layouts.get(key)
        if bt is None:
            bt = torch.tensor(np.repeat(np.asarray(ft, np.int32), B), device=dev)
            self._fast_layouts[key] = bt
        D = next(iter(self.deployment.metas.values())).dim
        self._segs_for(ft, fo, B, D)   # host -> device descriptor copy before capture
        c = self.cache
        if self._views is None or self._views[0] is not step:
            self._views = (step, [step.scalars_tensor(k) for k in range(step.n_slots)], c.scalars_tensor())
        stage_limit = max(0, int(self.params.admit_per_batch)) if self.params.adaptive_cache else 0
        do_maint = self.tracker is not None and self.policy is not None and self.params.adaptive_cache
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                sm = sample_major_starts(offsets, B, F)
                lay = CsrLayout(indices, offsets, bt, sm, None, [], None, None, None, B)
                out = torch.empty((B, F * D), dtype=torch.float32, device=dev)
                cnt = torch.empty((4, max(n_bags, 1)), dtype=torch.int32, device=dev)
                # K4 beside the step on a side stream (default), or after it on
                # the capture stream at full occupancy (FX_K4_SERIAL=1, A/B)
                serial = os.environ.get("FX_K4_SERIAL") == "1"
                side = self._pool_stream
                if not serial:
                    side.wait_stream(cap)
                    with torch.cuda.stream(side):
                        self._pool_sample_major(lay, out, ft, fo, B)
                step.start(0, bt, indices, offsets, sm, n_bags, nnz, self.params.pushdown_threshold, cnt[0], cnt[1],
                           cnt[2], cnt[3])
                step.offer(0)
                if do_maint:
                    step.maintain(0, stage_limit, True)
                step.join()
                if serial:
                    self._pool_sample_major(lay, out, ft, fo, B, share=False)
                else:
                    cap.wait_stream(side)
                snap = torch.cat([self._views[1][0], self._views[2]])
        torch.cuda.current_stream(dev).wait_stream(cap)
        return RankerGraph(self, g, out, cnt, snap, (indices, offsets, ft, fo, B), do_maint, step)

    def _fail(self, rec, err: int, err_at: int):
        from .step import ERR_BAD_INDEX, BatchStep
        if rec.get("tracker_before") is not None and self.tracker is not None:
            win, lvl = rec["tracker_before"]
            self.tracker.window.clear()
            self.tracker.window.extend(win)
            self._last_level = lvl
        if err == ERR_BAD_INDEX:
            raise self._validation_error(rec, err_at)
        BatchStep.raise_error(err, f"batch {rec.get('batch_id')}: ")

    def _validation_error(self, rec, err_at: int):
        """The reference's message for the first bad index in (lookup,
        feature, position) order (ranker.py:184-193)."""
        pos = err_at & 0xFFFFFFFF
        host = rec.get("host")
        if host is not None:
            try:
                host()
            except LookupValidationError as e:
                return e
        lay = rec.get("lay")
        if lay is None:
            return LookupValidationError(f"batch {rec.get('batch_id')}: index out of range")
        offs = lay.offsets.cpu().numpy()
        b = int(np.searchsorted(offs, pos, side="right") - 1)
        t = int(lay.bag_table[b].item())
        index = int(lay.indices[pos].item())
        n = self.deployment.meta(t).num_rows if t in self.deployment.metas else 0
        fs = rec.get("feature_shape")
        li = (b % fs[2]) if fs is not None else int(lay.perm[b] // max(1, len(lay.segs)))
        return LookupValidationError(f"batch {rec.get('batch_id')}, lookup {li}: index {index} out of "
                                     f"range [0,{n}) for table {t}")

    def _resolve(self) -> None:
        """[sync] turn every pending batch's device snapshot into BatchMetrics
        (and raise the first deferred device error)."""
        if not self._pending:
            return
        from .cache import _SC
        from .step import IDX, SCALARS
        pend, self._pending = self._pending, []
        pend[-1]["ev1"].synchronize()
        snaps = torch.stack([p["snap"] for p in pend]).cpu().numpy()
        ns = len(SCALARS)
        for p, row in zip(pend, snaps):
            ss, cs = row[:ns], row[ns:]
            if ss[IDX["err"]]:
                self._fail(p, int(ss[IDX["err"]]), int(ss[IDX["err_at"]]))
            entries = int(cs[_SC.index("entries")])
            m = BatchMetrics(
                batch_id=p["batch_id"], size=p["size"],
                started_at=self._epoch_ev.elapsed_time(p["ev0"]) / 1e3,
                latency=p["ev0"].elapsed_time(p["ev1"]) / 1e3,
                subrequests=int(ss[IDX["b_groups"]]),
                cache_hits=int(ss[IDX["b_hits"]]), cache_misses=int(ss[IDX["b_misses"]]),
                pushdown_groups=int(ss[IDX["b_pd_groups"]]), pushdown_rows=int(ss[IDX["b_pd_rows"]]),
                raw_rows=int(ss[IDX["b_raw_rows"]]), load_level=p["level"],
                # ranker.py:397-399: `if self.cache` is False while the cache is empty
                cache_budget=int(cs[_SC.index("budget")]) if entries else None,
                cache_used=int(cs[_SC.index("used")]) if entries else None)
            self.batch_metrics.append(m)
            cb = p.get("on_resolved")
            if cb is not None:
                cb(p, m)
        # keep the sketch table roomy enough for the next batches' new keys
        # (the fused step cannot grow it mid-stream)
        live = int(snaps[-1][ns + _SC.index("sketch_live")])
        st = self._step
        if st is not None and not self._inflight and (live + 1.5 * st.max_nnz) * 10 > self.cache.capacity()["sketch"] * 7:
            self.cache._reserve_sketch(2 * st.max_nnz + live)
            if self.cache.capacity()["sketch"] > st.tk_cap:
                self._step = None
                self._get_step(st.max_nnz, st.max_bags)   # rebuilt now, not inside a later batch

    def stream_host(self, host_batches, feature_tables, feature_ops, batch_size: int, depth: int = 3,
                    first_batch_id: int = 0, graphs: bool = True):
        """End-to-end batched API over HOST buffers: pinned host CSR batches
        (indices, offsets) in -> pinned host pooled [B, F*D] f32 out, in order.
        Three streams overlap the H2D of batch k+1, the Ranker batch k and the
        D2H of batch k-1. With `graphs` (pipeline_depth 1) a batch is a replay
        of one of two captured graphs (ping-pong over two static input / output
        buffer sets, Ranker.capture_csr), so the host only enqueues copies and
        a replay; a batch of another size runs eagerly. A yielded host tensor
        stays valid until the generator is advanced again (copy it to keep it)."""
        if not getattr(self, "_fast", False):
            raise ConfigError("stream_host needs the fused step (one full shard per table, one row size)")
        dev = self.device
        ft, fo, B = tuple(feature_tables), tuple(feature_ops), int(batch_size)
        D = next(iter(self.deployment.metas.values())).dim
        use_graphs = graphs and int(self.params.pipeline_depth) == 1
        cur = torch.cuda.current_stream(dev)
        nout = depth + 1
        # streams, device input slots, graphs and pinned outputs persist
        # across calls (pinned allocation and capture are slow)
        key = (depth, ft, fo, B, D)
        st = getattr(self, "_host_state", {}).get(key)
        if st is None:
            st = dict(streams=(torch.cuda.Stream(dev), torch.cuda.Stream(dev)), idx=[None] * depth,
                      offs=[torch.empty(len(ft) * B + 1, dtype=torch.int64, device=dev) for _ in range(depth)],
                      outs=[torch.empty((B, len(ft) * D), dtype=torch.float32, pin_memory=True)
                            for _ in range(nout)], graphs=None, gnnz=None)
            self._host_state = {key: st}
        s_in, s_out = st["streams"]
        idx_d, offs_d, outs_h = st["idx"], st["offs"], st["outs"]
        free = [None] * depth          # the batch that read input slot k is done
        done = [None] * nout           # D2H of output slot k finished
        gout_free = [None, None]       # D2H of a graph's static output finished
        queue = []
        for k, (idx_h, offs_h) in enumerate(host_batches):
            nnz = int(idx_h.numel())
            graphed = use_graphs and (st["gnnz"] in (None, nnz))
            sl = (k % 2) if graphed else k % depth
            if graphed and st["graphs"] is None:
                self.sync()
                gi = [torch.empty(max(nnz, 1), dtype=idx_h.dtype, device=dev) for _ in range(2)]
                go = [torch.empty(len(ft) * B + 1, dtype=torch.int64, device=dev) for _ in range(2)]
                st["graphs"] = [self.capture_csr(gi[i], go[i], ft, fo, B) for i in range(2)]
                st["gnnz"] = nnz
            if graphed and (st["graphs"][0].step is not self._step or not self.cache._queue_valid_host()):
                self.sync()
                self.reserve(nnz, len(ft) * B)
                self._step.prepare()
                st["graphs"] = [self.capture_csr(g.inputs[0], g.inputs[1], ft, fo, B) for g in st["graphs"]]
            if not graphed and (idx_d[sl] is None or idx_d[sl].numel() < nnz):
                idx_d[sl] = torch.empty(max(nnz, 1), dtype=idx_h.dtype, device=dev)
            if len(queue) >= depth:    # output slot reuse: hand the oldest result out first
                j, ev = queue.pop(0)
                ev.synchronize()
                yield outs_h[j % nout]
            if graphed:
                g = st["graphs"][sl]
                idx_dev, offs_dev = g.inputs[0], g.inputs[1]
            else:
                idx_dev, offs_dev = idx_d[sl][:nnz], offs_d[sl]
            with torch.cuda.stream(s_in):
                fr = (g.__dict__.get("free_ev") if graphed else free[sl])
                if fr is not None:
                    s_in.wait_event(fr)
                idx_dev.copy_(idx_h, non_blocking=True)
                offs_dev.copy_(offs_h, non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            cur.wait_event(ev_in)
            if graphed:
                if gout_free[sl] is not None:
                    cur.wait_event(gout_free[sl])   # its static output was copied out
                out = g.replay(batch_id=first_batch_id + k)
                fe = torch.cuda.Event()
                fe.record(cur)
                g.free_ev = fe
            else:
                out, _ = self.execute_csr(idx_dev, offs_dev, ft, fo, B, batch_id=first_batch_id + k, sync=False)
                fe = torch.cuda.Event()
                fe.record(cur)
                free[sl] = fe
            so = k % nout
            with torch.cuda.stream(s_out):
                s_out.wait_event(fe)
                if not graphed:
                    out.record_stream(s_out)
                outs_h[so].copy_(out, non_blocking=True)
                done[so] = torch.cuda.Event()
                done[so].record(s_out)
            if graphed:
                gout_free[sl] = done[so]
            queue.append((k, done[so]))
        while queue:
            j, ev = queue.pop(0)
            ev.synchronize()
            yield outs_h[j % nout]
        self.sync()

    def sync(self) -> None:
        """Finish every in-flight batch and resolve deferred metrics / errors."""
        while self._inflight:
            self._fast_finish()
        self._resolve()

    # -- driving ----------------------------------------------------------------

    def run_trace(self, trace_batches: list) -> None:
        """Closed-loop replay keeping up to `pipeline_depth` batches in flight
        (ranker.py:161-182): batch k+depth starts (apply_pending + probes)
        only after batch k finished (offers + maintenance), so with depth d
        the phases run S0..S(d-1) F0 Sd F1 ... — the reference's order when
        batches finish in arrival order (one server, FIFO)."""
        depth = max(1, int(self.params.pipeline_depth))
        if depth > 1 and self.cache is not None and not getattr(self, "_fast", False):
            raise ConfigError("pipeline_depth > 1 with a cache needs the fused step (one full shard per table on "
                              "this GPU, one row size, no pooled-result keyspace); the staged pipeline runs batches "
                              "one at a time and would not reproduce the reference's interleaving")
        if not getattr(self, "_fast", False) or depth == 1:
            for b in trace_batches:
                self._run_batch(b)
            return
        self.reserve(max(sum(len(f.indices) for lk in b.lookups for f in lk.features) for b in trace_batches),
                     max(sum(len(lk.features) for lk in b.lookups) for b in trace_batches))
        for b in trace_batches:
            for lookup in b.lookups:
                for f in lookup.features:
                    self.deployment.meta(f.table_id)
            if self._admission_needs_resize(b.size):
                raise ConfigError("pipeline_depth > 1 needs an admission check that never resizes the cache "
                                  "(MemoryModel capacity >= NN bytes + budget)")
            lay = pack_batch(b, self.device)
            rec = self._fast_start(lay, b.size, b.batch_id, host=lambda b=b: self._raise_validation(b))
            rec["on_resolved"] = lambda p, m, b=b: self._emit_fast(b, p)
            if len(self._inflight) >= depth:
                self._fast_finish()
        self.sync()

    def execute_batch(self, batch: Batch) -> list:
        self._run_batch(batch)
        return self.results.get(batch.batch_id, [])

    # -- pipeline ---------------------------------------------------------------

    def _raise_validation(self, batch: Batch):
        for li, lookup in enumerate(batch.lookups):
            for f in lookup.features:
                n = self.deployment.meta(f.table_id).num_rows
                for index in f.indices:
                    if not (0 <= index < n):
                        raise LookupValidationError(f"batch {batch.batch_id}, lookup {li}: index {index} out of "
                                                    f"range [0,{n}) for table {f.table_id}")
        raise InvariantError("device validation flagged an index the host check accepts")

    def _admission_check(self, batch: Batch) -> None:
        self._admission_check_size(batch.size, batch.batch_id)

    def _admission_check_size(self, size: int, batch_id: int) -> None:
        if self.cache is None or self.policy is None:
            return
        model = self.policy.model
        need = model.nn_bytes(size)
        if need > model.gpu_capacity_bytes:
            raise CapacityError(f"batch {batch_id} (size {size}) needs {need} NN bytes, "
                                f"capacity {model.gpu_capacity_bytes}")
        budget = self.cache.budget_bytes
        if need + budget <= model.gpu_capacity_bytes:
            return
        if not self.params.adaptive_cache:
            raise CapacityError(f"batch {batch_id} (size {size}): NN {need} bytes plus fixed cache "
                                f"{budget} exceeds capacity {model.gpu_capacity_bytes}")
        self.cache.resize(target_cache_bytes(model, size), fetcher=None)

    def _run_batch(self, batch: Batch) -> None:
        for lookup in batch.lookups:
            for f in lookup.features:
                self.deployment.meta(f.table_id)
        lay = pack_batch(batch, self.device)
        if getattr(self, "_fast", False) and not self._admission_needs_resize(batch.size):
            self.sync()
            rec = self._fast_start(lay, batch.size, batch.batch_id, host=lambda: self._raise_validation(batch))
            rec["on_resolved"] = lambda p, m: self._emit_fast(batch, p)
            self.sync()
            return
        self.sync()
        res, t = self._timed_pipeline(lay, batch.size, batch.batch_id, lambda: self._raise_validation(batch))
        self._emit(batch, lay, *res, times=t)

    def _timed_pipeline(self, lay, size, batch_id, bad):
        """The staged pipeline between two device events on the current
        stream: (results, (started_at, latency)) in seconds, started_at from
        the Ranker's first batch (BatchMetrics, ranker.py:60-72)."""
        if self._epoch_ev is None:
            self._epoch_ev = torch.cuda.Event(enable_timing=True)
            self._epoch_ev.record()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        res = self._pipeline(lay, size, batch_id, bad)
        ev1.record()
        ev1.synchronize()
        return res, (self._epoch_ev.elapsed_time(ev0) / 1e3, ev0.elapsed_time(ev1) / 1e3)

    def _emit_fast(self, batch: Batch, rec) -> None:
        """LookupResults of a fused-step batch (metrics already appended)."""
        cnt = rec["cnt"].cpu().numpy().astype(np.int64)
        lay = rec["lay"]
        n_bags = len(lay.perm)
        m = self.batch_metrics.pop()
        self._emit(batch, lay, rec["out"], torch.from_numpy(cnt[0, :n_bags]), torch.from_numpy(cnt[1, :n_bags]),
                   torch.from_numpy(cnt[2, :n_bags]), torch.from_numpy(cnt[3, :n_bags]), rec["nnz"], m.subrequests,
                   metrics=m)

    def execute_csr(self, indices: torch.Tensor, offsets: torch.Tensor, feature_tables, feature_ops,
                    batch_size: int, batch_id: int = 0, sync: bool = True):
        """Batched front end (no per-feature Python objects): table-major CSR
        in (bag = f*B + s), pooled [B, F*D] f32 + per-bag counter tensors out.
        Same pipeline, cache semantics and BatchMetrics as execute_batch.

        On the fused step (`sync=False`) nothing waits for the device: the
        batch's BatchMetrics and any deferred error (bad index, capacity) are
        resolved at the next `sync()` / `sync=True` call."""
        for t in feature_tables:
            self.deployment.meta(t)
        if getattr(self, "_fast", False) and not self._admission_needs_resize(batch_size):
            return self._execute_csr_fast(indices, offsets, tuple(feature_tables), tuple(feature_ops), batch_size,
                                          batch_id, sync)
        self.sync()
        lay = pack_csr(indices, offsets, feature_tables, feature_ops, batch_size, self.device)

        def bad():
            raise LookupValidationError(f"batch {batch_id}: index out of range (CSR batch)")
        (out, hits_bag, pd_groups, pd_rows, raw_rows, nnz, n_groups), (t0, lat) = self._timed_pipeline(
            lay, batch_size, batch_id, bad)
        F, B = len(feature_tables), batch_size
        dims = {self.deployment.meta(t).dim for t in feature_tables}
        D = out.shape[1]
        pooled = out.view(F, B, D).transpose(0, 1).reshape(B, F * D) if len(dims) == 1 else out
        c = self.cache
        hits = int(hits_bag.sum()) if c is not None else 0
        self.batch_metrics.append(BatchMetrics(
            batch_id=batch_id, size=batch_size, started_at=t0, latency=lat, subrequests=n_groups,
            cache_hits=hits, cache_misses=(nnz - hits) if c is not None else 0,
            pushdown_groups=int(pd_groups.sum()), pushdown_rows=int(pd_rows.sum()), raw_rows=int(raw_rows.sum()),
            load_level=self._last_level, cache_budget=(c.budget_bytes if c else None),
            cache_used=(c.used_bytes if c else None)))
        return pooled, dict(cache_hits=hits_bag, pushdown_groups=pd_groups, pushdown_rows=pd_rows,
                            raw_rows=raw_rows)

    def _execute_csr_fast(self, indices, offsets, feature_tables, feature_ops, B, batch_id, sync):
        dev = self.device
        F = len(feature_tables)
        key = (feature_tables, B)
        bt = self._fast_layouts.get(key)
        if bt is None:
            bt = torch.tensor(np.repeat(np.asarray(feature_tables, np.int32), B), device=dev)
            self._fast_layouts[key] = bt
        idx = indices if indices.dtype in (torch.int32, torch.int64) else indices.long()
        offs = offsets if offsets.dtype == torch.int64 else offsets.long()
        if offs.numel() != F * B + 1:
            raise ConfigError("offsets must describe batch_size * n_features table-major bags")
        lay = CsrLayout(idx, offs, bt, sample_major_starts(offs, B, F), None, [], None, None, None, B)
        rec = self._fast_start(lay, B, batch_id, feature_shape=(feature_tables, feature_ops, B))
        depth = max(1, int(self.params.pipeline_depth))
        while len(self._inflight) >= depth:
            self._fast_finish()
        if sync:
            self.sync()
        cnt = rec["cnt"]
        return rec["out"], dict(cache_hits=cnt[0], pushdown_groups=cnt[1], pushdown_rows=cnt[2], raw_rows=cnt[3])

    def _pipeline(self, lay: CsrLayout, n_lookups: int, batch_id: int, raise_validation):
        dev = self.device
        nnz = int(lay.indices.numel())
        n_bags = len(lay.perm)
        # 1. ingress validation + routing (K1)
        self._mark("route")
        self._status.reset()
        dest, _ = self.routing.route_csr(lay.bag_table, lay.indices, lay.offsets, status=self._status)
        code, _ = self._status.read()
        if code:
            raise_validation()
        cache = self.cache
        # 2. pending admissions, capacity gate
        self._mark("apply_pending")
        if cache is not None:
            cache.apply_pending_admissions()
        self._admission_check_size(n_lookups, batch_id)
        full_nnz = nnz
        lens_full = lay.offsets[1:] - lay.offsets[:-1]
        pooled = None
        n_ticks = nnz
        if cache is not None and cache.pooled_results_enabled and n_bags:
            # 2b. pooled-result probe per bag (ranker.py:238-245), then only the
            # residual bags go through row probes, pooling and offers
            self._mark("pooled_probe")
            pooled, lay, dest, n_ticks = self._pooled_probe(lay, dest, lens_full, n_bags)
            nnz = int(lay.indices.numel())
        # 3. dedup + probe (K2, K3)
        self._mark("dedup_probe")
        hit_occ = torch.zeros(nnz, dtype=torch.bool, device=dev)
        dd = None
        self._occ_slot = None
        if cache is not None and nnz:
            dd = self._dedup(lay.bag_table, lay.indices, lay.offsets, lay.sm_start, nnz)
            slot = torch.empty(max(dd.n_uniq, 1), dtype=torch.int32, device=dev)
            last = dd.last_ord if pooled is None else pooled[5][dd.last_ord]
            cache.probe_unique(dd.uniq, dd.mult, last, None, n_ticks, slot, n_uniq_host=dd.n_uniq)
            self._occ_slot = slot[dd.inverse.long()]
            hit_occ = self._occ_slot >= 0
        elif cache is not None and n_ticks:
            cache.advance_tick(n_ticks)
        # 4. miss groups per (bag, server) and the pushdown plan
        self._mark("plan")
        lens_tm = lay.offsets[1:] - lay.offsets[:-1]
        bag_of_occ = torch.repeat_interleave(torch.arange(n_bags, device=dev), lens_tm)
        n_srv = len(self._server_ids)
        srv_occ = self._shard_server_dev[dest.long()] if nnz else torch.zeros(0, dtype=torch.int64, device=dev)
        miss = ~hit_occ
        grp = torch.zeros(n_bags * n_srv, dtype=torch.int64, device=dev)
        if nnz:  # misses per (bag, server); hits add 0 (no host sync for a mask count)
            grp.index_add_(0, bag_of_occ * n_srv + srv_occ, miss.to(torch.int64))
        grp = grp.view(n_bags, n_srv)
        thr = self.params.pushdown_threshold
        if thr is None:
            push = torch.zeros_like(grp, dtype=torch.bool)
        else:
            if thr < 2:
                from .errors import EmbServeError
                raise EmbServeError(f"pushdown threshold must be >= 2, got {thr}")
            push = grp >= thr
        hits_bag = torch.zeros(n_bags, dtype=torch.int64, device=dev)
        if nnz:
            hits_bag.index_add_(0, bag_of_occ, hit_occ.long())
        if pooled is not None:  # a pooled hit counts every index as a cache hit (ranker.py:242-243)
            hits_bag += torch.where(pooled[1], lens_full, torch.zeros_like(lens_full))
        pd_groups = push.sum(1)
        pd_rows = (grp * push).sum(1)
        raw_rows = (grp * (~push)).sum(1)
        n_groups = int((grp > 0).sum())
        # 5. pooled vectors: per-shard f64 partials of the misses + cache rows as raw
        self._mark("pool")
        out = self._pool(lay, dest, hit_occ, dd, nnz, n_bags)
        if pooled is not None:
            self._pooled_finish(lay, pooled, out, n_bags)
        self._mark("offers")
        # 6. offers: raw-fetched misses, first raw occurrence order
        if cache is not None and nnz:
            raw_occ = miss & ~push.view(-1)[bag_of_occ * n_srv + srv_occ]
            # first raw occurrence (sample-major ordinal) of every unique key; keys
            # without a raw occurrence keep BIG (masked scatter: one host sync, for the count)
            BIG = 1 << 62
            ords = lay.sm_start[bag_of_occ] + (torch.arange(nnz, device=dev) - lay.offsets[bag_of_occ])
            big = torch.full((dd.n_uniq,), BIG, dtype=torch.int64, device=dev)
            big.scatter_reduce_(0, dd.inverse.long(), torch.where(raw_occ, ords, torch.full_like(ords, BIG)),
                                reduce="amin")
            cand = torch.nonzero(big < BIG).view(-1)
            if cand.numel():
                order = torch.argsort(big[cand])
                keys = dd.uniq[cand[order]].contiguous()
                cache.offer_keys(keys, int(keys.numel()))
        # 7. maintenance
        self._mark("maintenance")
        self._maintenance_size(n_lookups)
        self._mark("end")
        self._flush_marks()
        # results (sample-major)
        return out, hits_bag, pd_groups, pd_rows, raw_rows, full_nnz, n_groups

    def _pooled_probe(self, lay: CsrLayout, dest, lens, n_bags):
        """Fingerprint every bag, find its pooled entry, apply the hits'
        recency at their tick positions, and cut the hit bags out of the CSR.
        Ticks run in sample-major order: one per pooled_get, then one per row
        probe of a missed bag (ranker.py:238-251)."""
        from .cache import bag_fingerprints
        dev = self.device
        cache = self.cache
        ops = torch.empty(n_bags, dtype=torch.int32, device=dev)
        for (t, opc, b0, b1) in lay.segs:
            ops[b0:b1] = opc
        ka, kb = bag_fingerprints(lay.bag_table, ops, lay.indices, lay.offsets)
        pslot = torch.empty(n_bags, dtype=torch.int32, device=dev)
        cache.pooled_find(ka, kb, pslot)
        phit = pslot >= 0
        cost = 1 + torch.where(phit, torch.zeros_like(lens), lens)       # table-major bags
        perm = torch.as_tensor(lay.perm, dtype=torch.int64, device=dev)   # tm bag -> sm bag
        cost_sm = torch.empty_like(cost)
        cost_sm[perm] = cost
        pos = (torch.cumsum(cost_sm, 0) - cost_sm)[perm]                  # tick offset of each bag's pooled_get
        cache.pooled_touch(pslot, pos)
        keep_bag = ~phit
        lens_r = torch.where(keep_bag, lens, torch.zeros_like(lens))
        offs_r = torch.zeros(n_bags + 1, dtype=torch.int64, device=dev)
        offs_r[1:] = torch.cumsum(lens_r, 0)
        keep_occ = torch.repeat_interleave(keep_bag, lens)
        # dedup wants dense sample-major ordinals of the residual occurrences;
        # tick_of[ord] maps them back to the row probe's tick offset
        lr_sm = torch.empty_like(lens_r)
        lr_sm[perm] = lens_r
        smc = (torch.cumsum(lr_sm, 0) - lr_sm)[perm]
        nnz_r = int(offs_r[-1])
        bag_occ = torch.repeat_interleave(torch.arange(n_bags, device=dev), lens_r)
        within = torch.arange(nnz_r, device=dev) - offs_r[bag_occ]
        tick_of = torch.empty(max(nnz_r, 1), dtype=torch.int64, device=dev)
        tick_of[smc[bag_occ] + within] = pos[bag_occ] + 1 + within
        rl = CsrLayout(lay.indices[keep_occ], offs_r, lay.bag_table, smc, lay.perm, lay.segs, lay.lens_sm,
                       lay.bag_lookup_sm, lay.host_idx_sm, lay.n_lookups)
        n_ticks = int(cost.sum())
        return (pslot, phit, ka, kb, perm, tick_of), rl, dest[keep_occ], n_ticks

    def _pooled_finish(self, lay: CsrLayout, pooled, out, n_bags):
        """Hit bags take the cached vector; every other bag is put, in
        sample-major (finish) order, before the row offers (ranker.py:401-414)."""
        pslot, phit, ka, kb, perm, _ = pooled
        cache = self.cache
        if self.profile:
            self.last_pooled_hits = int(phit.sum())
        cache.read_slots(pslot, out)
        order_tm = torch.argsort(perm)                # tm bags in sample-major order
        put_tm = order_tm[~phit[order_tm]]
        if put_tm.numel():
            dims = [self.deployment.meta(t).dim for t, *_ in lay.segs]
            if len(set(dims)) != 1:
                raise ConfigError("pooled-result keyspace with mixed table dims in one batch is not supported")
            cache.pooled_put_many(ka[put_tm].contiguous(), kb[put_tm].contiguous(), out, dims[0] * 4, sel=put_tm)
        cache.check_state()

    def _pool(self, lay: CsrLayout, dest, hit_occ, dd, nnz, n_bags) -> torch.Tensor:
        dims = {self.deployment.meta(t).dim for t, *_ in lay.segs}
        if self._single_shard and len(dims) == 1 and (self.cache is None or not self.hits_from_cache):
            return self._pool_fused(lay, n_bags)
        return self._pool_partials(lay, dest, hit_occ, dd, nnz, n_bags)

    def _pool_fused(self, lay: CsrLayout, n_bags, out=None) -> torch.Tensor:
        """One K4 launch over the whole batch (f64 accumulate, one rounding)."""
        dev = self.device
        dims = {self.deployment.meta(t).dim for t, *_ in lay.segs}
        D = max(dims) if dims else 1
        if out is None:
            out = torch.zeros((n_bags, D), dtype=torch.float32, device=dev)
        if n_bags == 0:
            return out
        for dim in sorted(dims):
            segs = []
            for (t, opc, b0, b1) in lay.segs:
                if self.deployment.meta(t).dim != dim:
                    continue
                tab, start, end, _, _ = self._table_shard[t]
                segs.append(_lib.FxSegment(tab.data_ptr(), start, end, b0, b1, out.data_ptr() + b0 * D * 4, D,
                                           tab.stride(0), dim, opc))
            seg_dev = make_segments(self._cover_out(segs, n_bags, D, out), dev)
            _lib.check(_lib.lib.fx_gather_pool(seg_dev.data_ptr(), seg_dev.numel() // _lib.SEGMENT_BYTES, dim,
                                               lay.indices.data_ptr(), _lib.FX_IDX_I64, lay.offsets.data_ptr(),
                                               n_bags, _lib.FX_OUT_F32, None, self._status.err.data_ptr(),
                                               _lib.FX_E_ROUTING_VIOLATION, self._status.code.data_ptr(),
                                               _lib.stream_ptr()), "fused pool")
        return out

    @staticmethod
    def _cover_out(segs, n_bags, D, out):
        """Cover [0, n_bags) with segments; gaps (bags of another dim) get a
        scratch segment whose output lands in a throw-away row range."""
        res, cursor = [], 0
        for sg in sorted(segs, key=lambda s: s.bag_begin):
            if sg.bag_begin > cursor:
                raise InvariantError("mixed-dim batches take the partial path")
            res.append(sg)
            cursor = sg.bag_end
        if cursor < n_bags:
            raise InvariantError("mixed-dim batches take the partial path")
        return res

    def _pool_partials(self, lay: CsrLayout, dest, hit_occ, dd, nnz, n_bags) -> torch.Tensor:
        """Partial pool per shard (K4 FX_OUT_F64_PARTIAL over that shard's miss
        occurrences, bucketed in (bag, position) order by fx_bucket), then K5
        folds partials in ascending shard order plus cache rows in position order."""
        dev = self.device
        dims = {self.deployment.meta(t).dim for t, *_ in lay.segs}
        D = max(dims) if dims else 1
        n_sh = len(self._shards)
        out = torch.empty((n_bags, D), dtype=torch.float32, device=dev)
        if n_bags == 0:
            return out
        dest_m = torch.where(hit_occ, torch.full_like(dest, n_sh), dest) if nnz else dest
        perm = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        dcount = torch.empty(n_sh + 1, dtype=torch.int64, device=dev)
        bcount = torch.empty((n_sh + 1) * n_bags, dtype=torch.int32, device=dev)
        need = ctypes.c_size_t(0)
        _lib.check(_lib.lib.fx_bucket(None, nnz, None, n_bags, n_sh + 1, None, None, None, None, ctypes.byref(need),
                                      None), "bucket")
        ws = torch.empty(max(need.value, 1), dtype=torch.uint8, device=dev)
        _lib.check(_lib.lib.fx_bucket(dest_m.data_ptr() if nnz else None, nnz, lay.offsets.data_ptr(), n_bags, n_sh + 1,
                                      perm.data_ptr(), dcount.data_ptr(), bcount.data_ptr(), ws.data_ptr(),
                                      ctypes.byref(need), _lib.stream_ptr()), "bucket")
        dc = dcount.cpu().numpy()
        bcount = bcount.view(n_sh + 1, n_bags)
        starts = np.concatenate([[0], np.cumsum(dc)])
        sorted_idx = lay.indices[perm[:nnz]] if nnz else lay.indices
        partials, counts = [], []
        for sid, (tab, start, end, server, table) in enumerate(self._shards):
            if dc[sid] == 0:
                continue
            offs = torch.zeros(n_bags + 1, dtype=torch.int64, device=dev)
            offs[1:] = torch.cumsum(bcount[sid].long(), 0)
            idx_s = sorted_idx[starts[sid]:starts[sid + 1]]
            part = torch.zeros((n_bags, D), dtype=torch.float64, device=dev)
            cnt = torch.zeros(n_bags, dtype=torch.int32, device=dev)
            segs = []
            for (t, opc, b0, b1) in lay.segs:
                if t != table:
                    continue
                segs.append(_lib.FxSegment(tab.data_ptr(), start, end, b0, b1, part.data_ptr() + b0 * D * 8, D,
                                           tab.stride(0), tab.shape[1], 0))
            if not segs:
                continue
            # bags of other tables have zero rows for this shard; give them a dummy segment range
            seg_dev = make_segments(self._cover(segs, n_bags, tab, start, end, part, D), dev)
            _lib.check(_lib.lib.fx_gather_pool(seg_dev.data_ptr(), seg_dev.numel() // _lib.SEGMENT_BYTES,
                                               tab.shape[1], idx_s.data_ptr(), _lib.FX_IDX_I64, offs.data_ptr(),
                                               n_bags, _lib.FX_OUT_F64_PARTIAL, cnt.data_ptr(),
                                               self._status.err.data_ptr(), _lib.FX_E_ROUTING_VIOLATION,
                                               self._status.code.data_ptr(), _lib.stream_ptr()), "partial pool")
            partials.append(part)
            counts.append(cnt)
        # cache-hit rows (raw vectors, position order)
        raw_off = raw_rows = None
        if nnz and bool(hit_occ.any()):
            hb = bcount[n_sh].long()
            raw_off = torch.zeros(n_bags + 1, dtype=torch.int64, device=dev)
            raw_off[1:] = torch.cumsum(hb, 0)
            hit_keys = (lay.bag_table.long()[torch.repeat_interleave(torch.arange(n_bags, device=dev),
                                                                     lay.offsets[1:] - lay.offsets[:-1])] << 40
                        | lay.indices)[perm[starts[n_sh]:starts[n_sh + 1]]]
            raw_rows = torch.zeros((hit_keys.numel(), self.cache.max_dim), dtype=torch.float32, device=dev)
            slot = torch.empty(hit_keys.numel(), dtype=torch.int32, device=dev)
            _lib.check(self.cache._L.fx_cache_lookup(self.cache._h, hit_keys.data_ptr(), hit_keys.numel(),
                                                     raw_rows.data_ptr(), self.cache.max_dim, slot.data_ptr(),
                                                     _lib.stream_ptr()), "cache rows")
            raw_rows = raw_rows[:, :D].contiguous()
        n_src = len(partials)
        ptrs = torch.tensor([p.data_ptr() for p in partials] or [0], dtype=torch.int64, device=dev)
        cptr = torch.tensor([c.data_ptr() for c in counts] or [0], dtype=torch.int64, device=dev)
        ops = torch.zeros(n_bags, dtype=torch.int32, device=dev)
        for (t, opc, b0, b1) in lay.segs:
            ops[b0:b1] = opc
        _lib.check(_lib.lib.fx_combine(ptrs.data_ptr(), 0, cptr.data_ptr(), n_src, D, _lib.ptr(raw_off),
                                       _lib.ptr(raw_rows), n_bags, D, 0, ops.data_ptr(), out.data_ptr(), D, None,
                                       _lib.stream_ptr()), "combine")
        return out

    @staticmethod
    def _cover(segs, n_bags, tab, start, end, part, D):
        """Extend a shard's segment list to cover [0, n_bags) (bags of other
        tables get empty ranges: their offsets are zero-length for this shard)."""
        out = []
        cursor = 0
        for sg in sorted(segs, key=lambda s: s.bag_begin):
            if sg.bag_begin > cursor:
                out.append(_lib.FxSegment(tab.data_ptr(), start, end, cursor, sg.bag_begin,
                                          part.data_ptr() + cursor * D * 8, D, tab.stride(0), tab.shape[1], 0))
            out.append(sg)
            cursor = sg.bag_end
        if cursor < n_bags:
            out.append(_lib.FxSegment(tab.data_ptr(), start, end, cursor, n_bags, part.data_ptr() + cursor * D * 8,
                                      D, tab.stride(0), tab.shape[1], 0))
        return out

    def _maintenance(self, batch: Batch) -> None:
        self._maintenance_size(batch.size)

    def _maintenance_size(self, size: int) -> None:
        c = self.cache
        if c is None or self.tracker is None or self.policy is None:
            return
        level = self.tracker.record_batch(size)
        self._last_level = level.value
        if not self.params.adaptive_cache:
            return
        rb = lambda t: self.deployment.meta(t).row_bytes
        fetcher = lambda t, i: self.deployment.get_row(t, i)
        budget = c.budget_bytes
        proposed = self.policy.propose(budget, level, self.tracker.windowed_value())
        if proposed != budget:
            c.resize(proposed, fetcher=fetcher, row_bytes_of=rb)
        if self.params.admit_per_batch > 0:
            c.stage_hot_admissions(fetcher, rb, limit=self.params.admit_per_batch)
        c.sketch.age()

    def _emit(self, batch, lay, out, hits_bag, pd_groups, pd_rows, raw_rows, nnz, n_groups, metrics=None,
              times=(0.0, 0.0)):
        n_bags = len(lay.perm)
        inv = np.empty(n_bags, dtype=np.int64)
        inv[lay.perm] = np.arange(n_bags)
        vec = out.cpu().numpy()
        hb = hits_bag.cpu().numpy()
        pg = pd_groups.cpu().numpy()
        pr = pd_rows.cpu().numpy()
        rr = raw_rows.cpu().numpy()
        results = []
        b_sm = 0
        tot = np.zeros(4, np.int64)
        for li, lookup in enumerate(batch.lookups):
            res = LookupResult()
            for f in lookup.features:
                b = inv[b_sm]
                dim = self.deployment.meta(f.table_id).dim
                res.vectors.append(vec[b, :dim].copy())
                res.cache_hits += int(hb[b])
                res.pushdown_groups += int(pg[b])
                res.pushdown_rows += int(pr[b])
                res.raw_rows += int(rr[b])
                b_sm += 1
            if res.cache_hits + res.pushdown_rows + res.raw_rows != lookup.total_indices():
                raise InvariantError(f"counter conservation broken on lookup {li}: {res.counters} vs "
                                     f"{lookup.total_indices()} indices")
            tot += (res.cache_hits, res.pushdown_groups, res.pushdown_rows, res.raw_rows)
            results.append(res)
        c = self.cache
        hits = int(tot[0]) if c is not None else 0
        misses = (nnz - hits) if c is not None else 0
        sub = n_groups  # one subrequest per (lookup, feature, server) group (ranker.py:275-301)
        if metrics is not None:
            if (metrics.cache_hits, metrics.pushdown_groups, metrics.pushdown_rows, metrics.raw_rows) != tuple(
                    int(x) for x in tot):
                raise InvariantError("fused step counters disagree with the per-bag counters")
            self.batch_metrics.append(metrics)
            if self.params.keep_results:
                self.results[batch.batch_id] = results
            return
        self.batch_metrics.append(BatchMetrics(
            batch_id=batch.batch_id, size=batch.size, started_at=times[0], latency=times[1], subrequests=sub,
            cache_hits=hits, cache_misses=misses, pushdown_groups=int(tot[1]), pushdown_rows=int(tot[2]),
            raw_rows=int(tot[3]), load_level=self._last_level,
            cache_budget=(c.budget_bytes if c else None), cache_used=(c.used_bytes if c else None)))
        if self.params.keep_results:
            self.results[batch.batch_id] = results


class RankerGraph:
    """A captured fused Ranker batch (Ranker.capture_csr). `out` / `counters`
    are static: they hold the last replay's pooled [B, F*D] vectors and per-bag
    counters until the next replay."""

    def __init__(self, rk, graph, out, cnt, snap, inputs, do_maint, step):
        self.rk, self.graph, self.out, self.cnt, self.snap = rk, graph, out, cnt, snap
        self.inputs = inputs
        self.do_maint = do_maint
        self.step = step  # the graph bakes this step's buffers in (kept alive)

    @property
    def counters(self) -> dict:
        c = self.cnt
        return dict(cache_hits=c[0], pushdown_groups=c[1], pushdown_rows=c[2], raw_rows=c[3])

    def replay(self, batch_id: int = 0) -> torch.Tensor:
        rk = self.rk
        idx, offs, ft, fo, B = self.inputs
        c = rk.cache
        if rk._step is not self.step or not c._queue_valid_host():
            raise ConfigError("the Ranker rebuilt its fused step or another cache call moved entries since "
                              "capture_csr: capture again")
        if rk._admission_needs_resize(B):
            raise ConfigError("the captured batch's admission check would resize the cache: run execute_csr")
        rec = dict(batch_id=batch_id, size=B, lay=None, host=None, feature_shape=(ft, fo, B))
        rec["tracker_before"] = (list(rk.tracker.window), rk._last_level) if rk.tracker is not None else None
        if rk.tracker is not None and rk.policy is not None:
            level = rk.tracker.record_batch(B)
            rk._last_level = level.value
            if rk.params.adaptive_cache and rk.policy.propose(c.budget_bytes, level,
                                                              rk.tracker.windowed_value()) != c.budget_bytes:
                # the graph bakes in "no budget change": undo and run this batch eagerly
                win, lvl = rec["tracker_before"]
                rk.tracker.window.clear()
                rk.tracker.window.extend(win)
                rk._last_level = lvl
                out, cnt = rk.execute_csr(idx, offs, ft, fo, B, batch_id=batch_id, sync=False)
                self.out.copy_(out)
                return self.out
        cur = torch.cuda.current_stream(rk.device)
        if rk._epoch_ev is None:
            rk._epoch_ev = torch.cuda.Event(enable_timing=True)
            rk._epoch_ev.record(cur)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(cur)
        self.graph.replay()
        ev1.record(cur)
        rec.update(ev0=ev0, ev1=ev1, snap=self.snap.clone(), level=rk._last_level)
        rk._pending.append(rec)
        return self.out


@dataclass
class EquivalenceReport:
    lookups_checked: int
    max_abs_diff: float
    max_tolerance_ratio: float

    @property
    def passed(self) -> bool:
        return self.max_tolerance_ratio <= 1.0


def flat_reference(deployment: Deployment, lookup: LookupRequest) -> list:
    """No cache, no pushdown: direct row reads pooled flat (ranker.py:458-465),
    computed on the GPU (K4 over the gathered rows)."""
    out = []
    for f in lookup.features:
        rows = torch.stack([deployment.get_row_device(f.table_id, i) for i in f.indices])
        out.append(pool_flat(rows, f.op).cpu().numpy())
    return out


def end_to_end_equivalence_check(deployment, batches, results, rel_tol=1e-5, abs_floor=1e-6) -> EquivalenceReport:
    checked, max_abs, max_ratio = 0, 0.0, 0.0
    for batch in batches:
        for lookup, result in zip(batch.lookups, results[batch.batch_id]):
            for ref, got in zip(flat_reference(deployment, lookup), result.vectors):
                diff = np.abs(ref.astype(np.float64) - got.astype(np.float64))
                bound = np.maximum(abs_floor, rel_tol * np.abs(ref.astype(np.float64)))
                max_abs = max(max_abs, float(diff.max(initial=0.0)))
                max_ratio = max(max_ratio, float((diff / bound).max(initial=0.0)))
            checked += 1
    return EquivalenceReport(checked, max_abs, max_ratio)
