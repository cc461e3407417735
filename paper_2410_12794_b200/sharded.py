"""Multi-GPU sharded lookup: one process per GPU, tables table-wise or
row-wise sharded in HBM across the ranks of one box, pooled results returned
to the requesting GPU over NCCL all-to-all (NVLink 5 / NVSwitch).

This replaces the reference's fan-out seam (ranker.py:263-347 _fan_out ->
VirtualTransport.post_subrequest -> _server_handler -> _on_response): a
"server" is a GPU rank, a subrequest is the slice of a requester's CSR batch
routed to that rank, and the response is pooled vectors (pushdown):

  requester: K1 fx_route (index -> owning rank) + fx_bucket (stable per-rank
             CSR, GroupItem.positions semantics)            routing.py:117-148
  C1:        all_to_all of per-destination counts, per-bag lengths, indices
  owner:     K4 gather+pool over its local shards: table-wise -> final f32
             (whole bag local, one rounding); row-wise -> f64 partial + count
             (PartialResult(sum, count), store.py:184-193)
  C2:        all_to_all of pooled rows back to the requester
  requester: table-wise -> placement into out[B, F*D];
             row-wise -> K5 fx_combine in ascending source rank (pooling.py:103-123)

Every rank runs the same per-GPU batch shape (weak scaling). The compute
steps live behind `FlexOps` (libflexemb kernels); the exchange protocol
itself is backend-agnostic torch.distributed (NCCL on GPUs; the CPU tests
run it under gloo with a test double for the ops).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigError, LookupValidationError, RoutingViolationError
from .store import ShardSpec


def tablewise_placement(table_rows, world: int):
    """Greedy balance of tables over ranks by row count (largest first);
    one shard per table (cfg4 placement)."""
    order = sorted(range(len(table_rows)), key=lambda t: -table_rows[t])
    load = [0] * world
    count = [0] * world
    owner = [0] * len(table_rows)
    for t in order:
        r = min(range(world), key=lambda i: (count[i], load[i], i))
        owner[t] = r
        load[r] += table_rows[t]
        count[r] += 1
    return [ShardSpec(t, 0, int(n), owner[t]) for t, n in enumerate(table_rows)]


def rowwise_placement(table_rows, world: int):
    """Each table split into min(world, rows) contiguous ranges, range k on
    rank k (cfg5 placement)."""
    specs = []
    for t, n in enumerate(table_rows):
        s = min(world, int(n))
        bounds = [int(round(i * n / s)) for i in range(s + 1)]
        for k in range(s):
            specs.append(ShardSpec(t, bounds[k], bounds[k + 1], k))
    return specs


class FlexOps:
    """Device compute of the sharded path, all in libflexemb kernels."""

    def __init__(self, metas: dict, placement, seed: int, rank: int, feature_tables, feature_ops, B: int, device,
                 ipc_shards: bool = False):
        """`ipc_shards`: allocate the local shards with cudaMalloc (fx_dev_alloc)
        so peers can map them (raw fetch over NVLink)."""
        from . import _lib
        from .store import table_block_device
        self._lib = _lib
        self.device = torch.device(device)
        self.rank = rank
        self.B = B
        self.ftab = tuple(feature_tables)
        self.fops = tuple(feature_ops)
        self.local = {}
        self.shard_bufs = {}
        for sp in placement:
            if sp.server_id == rank:
                D = metas[sp.table_id].dim
                out = None
                if ipc_shards:
                    buf = DevBuffer((sp.end - sp.start) * D * 4)
                    self.shard_bufs[sp.table_id] = buf
                    out = _cai_tensor(buf.ptr, (sp.end - sp.start, D), torch.float32, self.device)
                data = table_block_device(seed, sp.table_id, D, sp.start, sp.end, device=self.device, out=out)
                self.local[sp.table_id] = (data, sp.start, sp.end)
        n_t = max(metas) + 1
        route_off = np.zeros(n_t + 1, np.int64)
        starts, owners = [], []
        self.shard_list = []  # routing order (table, start): global shard ids
        for t in range(n_t):
            sh = sorted((s for s in placement if s.table_id == t), key=lambda s: s.start)
            route_off[t + 1] = route_off[t] + len(sh)
            starts += [s.start for s in sh]
            owners += [s.server_id for s in sh]
            self.shard_list += sh
        nrows = np.array([metas[t].num_rows if t in metas else 0 for t in range(n_t)], np.int64)
        dev = self.device
        self.route_off = torch.from_numpy(route_off).to(dev)
        self.starts = torch.tensor(starts, dtype=torch.int64, device=dev)
        self.owners = torch.tensor(owners, dtype=torch.int32, device=dev)
        self.nrows = torch.from_numpy(nrows).to(dev)
        self.bag_table = torch.tensor(np.repeat(np.array(self.ftab, np.int32), B), device=dev)
        self.status = _lib.Status(dev)        # requester-side ingress validation (K1)
        self.owner_status = _lib.Status(dev)  # owner-side: rows routed here that it does not host (K4)
        self._ws = None
        self._seg_cache = {}

    def route_bucket(self, indices, offsets, world: int):
        """-> (send_idx int32 in (dest, bag, pos) order, dcount int64[W], bcount int32[W, n_bags])."""
        L = self._lib
        dev = self.device
        n_bags = offsets.numel() - 1
        nnz = int(indices.numel())
        idx = indices.to(torch.int64) if indices.dtype != torch.int64 else indices
        dest = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        L.check(L.lib.fx_route(self.route_off.data_ptr(), self.starts.data_ptr(), self.owners.data_ptr(),
                               self.nrows.data_ptr(), self.bag_table.data_ptr(), idx.data_ptr(), L.FX_IDX_I64,
                               offsets.data_ptr(), n_bags, dest.data_ptr(), self.status.err.data_ptr(),
                               self.status.code.data_ptr(), L.stream_ptr()), "route")
        # an invalid index (flagged above, raised by check()) still needs a
        # destination so every rank's split sizes agree: rank 0, which then
        # records a routing violation instead of reading it
        dest.clamp_(min=0)
        need = ctypes.c_size_t(0)
        L.check(L.lib.fx_bucket(None, nnz, None, n_bags, world, None, None, None, None, ctypes.byref(need), None))
        if self._ws is None or self._ws.numel() < need.value:
            self._ws = torch.empty(max(need.value, 1), dtype=torch.uint8, device=dev)
        perm = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        dcount = torch.empty(world, dtype=torch.int64, device=dev)
        bcount = torch.empty(world * n_bags, dtype=torch.int32, device=dev)
        L.check(L.lib.fx_bucket(dest.data_ptr(), nnz, offsets.data_ptr(), n_bags, world, perm.data_ptr(),
                                dcount.data_ptr(), bcount.data_ptr(), self._ws.data_ptr(), ctypes.byref(need),
                                L.stream_ptr()), "bucket")
        return idx[perm[:nnz]].to(torch.int32), dcount, bcount.view(world, n_bags)

    def _segments(self, out, feats, partial):
        from .pooling import op_code
        from .store import make_segments
        L = self._lib
        key = (out.data_ptr(), partial, tuple(feats))
        seg = self._seg_cache.get(key)
        if seg is not None:
            return seg
        B = self.B
        D = out.shape[-1]
        esz = 8 if partial else 4
        segs = []
        for j, f in enumerate(feats):
            t = self.ftab[f]
            tp, rb, re = (self.local[t][0].data_ptr(), self.local[t][1], self.local[t][2]) if t in self.local \
                else (0, 0, 0)
            segs.append(L.FxSegment(tp, rb, re, j * B, (j + 1) * B, out.data_ptr() + j * B * D * esz, D, D, D,
                                    op_code(self.fops[f])))
        seg = make_segments(segs, self.device)
        self._seg_cache[key] = seg
        if len(self._seg_cache) > 128:
            self._seg_cache.pop(next(iter(self._seg_cache)))
        return seg

    def owner_pool(self, recv_idx, lens, feats, out, partial: bool, counts=None):
        """K4 over one requester's bags of `feats` (lens: int32 per bag)."""
        L = self._lib
        n = lens.numel()
        if n == 0:
            return
        offs = torch.zeros(n + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(lens.long(), 0, out=offs[1:])
        seg = self._segments(out, feats, partial)
        L.check(L.lib.fx_gather_pool(seg.data_ptr(), len(feats), out.shape[-1], recv_idx.data_ptr(), L.FX_IDX_I32,
                                     offs.data_ptr(), n, L.FX_OUT_F64_PARTIAL if partial else L.FX_OUT_F32,
                                     L.ptr(counts), self.owner_status.err.data_ptr(), L.FX_E_ROUTING_VIOLATION,
                                     self.owner_status.code.data_ptr(), L.stream_ptr()), "owner pool")

    def combine(self, parts, cnts, bag_ops, out):
        """K5: fold per-source f64 partials in ascending source rank."""
        L = self._lib
        W, n_bags, D = parts.shape
        ptrs = torch.tensor([parts[s].data_ptr() for s in range(W)], dtype=torch.int64, device=self.device)
        cptr = torch.tensor([cnts[s].data_ptr() for s in range(W)], dtype=torch.int64, device=self.device)
        L.check(L.lib.fx_combine(ptrs.data_ptr(), 0, cptr.data_ptr(), W, D, None, None, n_bags, D, 0, bag_ops.data_ptr(),
                                 out.data_ptr(), D, None, L.stream_ptr()), "combine")

    def check(self, batch=None, batch_id: int = 0):
        """[sync] Raise for a flagged index: LookupValidationError with the
        reference's message (ranker.py:184-193) when this rank's own batch
        held it (`batch` = (indices, offsets) of that batch), else
        RoutingViolationError (an owner was sent a row it does not host)."""
        code, pos = self.status.read()
        ocode, _ = self.owner_status.read()
        if not code and not ocode:
            return
        self.status.reset()
        self.owner_status.reset()
        if code:
            if batch is not None:
                # the reference rejects the first bad index in (lookup, feature,
                # position) order (ranker.py:184-193); the device flag holds the
                # first in CSR (feature-major) order, so rescan on the host
                idx, offs = batch
                offs_h = offs.cpu().numpy().astype(np.int64)
                idx_h = idx.cpu().numpy().astype(np.int64)
                nbag = offs_h.size - 1
                lens = np.diff(offs_h)
                bag_of = np.repeat(np.arange(nbag), lens)
                nrows = np.array([int(self.nrows[t].item()) for t in self.ftab], np.int64)
                f_of = bag_of // self.B
                bad = np.nonzero((idx_h < 0) | (idx_h >= nrows[f_of]))[0]
                if bad.size:
                    smp_of, fp = bag_of[bad] % self.B, f_of[bad]
                    first = bad[np.lexsort((bad, fp, smp_of))[0]]
                    f, smp = divmod(int(bag_of[first]), self.B)
                    t = self.ftab[f]
                    raise LookupValidationError(f"batch {batch_id}, lookup {smp}: index {int(idx_h[first])} "
                                                f"out of range [0,{int(nrows[f])}) for table {t}")
            raise LookupValidationError(f"batch {batch_id}: index out of range at CSR position {pos} "
                                        f"(rank {self.rank})")
        raise RoutingViolationError(f"rank {self.rank} was sent a row it does not host")


@dataclass
class ExchangeStats:
    c1_bytes_sent: int = 0
    c2_bytes_sent: int = 0
    calls: int = 0


class ShardedLookup:
    """Per-rank sharded lookup. `feature_tables` fixes the batch layout
    (feature f reads table feature_tables[f]); every rank submits batches of
    `batch_size` samples, table-major CSR (bag = f*B + s)."""

    def __init__(self, metas, placement, seed: int, feature_tables, feature_ops, batch_size: int, rank: int,
                 world: int, device, group=None, mode: str = "tablewise", ops=None):
        if mode not in ("tablewise", "rowwise"):
            raise ConfigError(f"unknown sharding mode {mode!r}")
        self.metas = {m.table_id: m for m in metas}
        self.rank, self.world = rank, world
        self.device = torch.device(device)
        self.group = group
        self.mode = mode
        self.B = batch_size
        self.ftab = tuple(feature_tables)
        self.fops = tuple(feature_ops)
        self.F = len(self.ftab)
        dims = {self.metas[t].dim for t in self.ftab}
        if len(dims) != 1:
            raise ConfigError("sharded lookup needs one embedding dim across features")
        self.D = dims.pop()
        per_rank = {}
        for sp in placement:
            if sp.server_id >= world:
                raise ConfigError(f"shard of table {sp.table_id} placed on rank {sp.server_id} >= world {world}")
            per_rank.setdefault((sp.server_id, sp.table_id), 0)
            per_rank[(sp.server_id, sp.table_id)] += 1
            if per_rank[(sp.server_id, sp.table_id)] > 1:
                raise ConfigError("one shard per table per rank")
        tab_owner = {}
        for sp in placement:
            tab_owner.setdefault(sp.table_id, set()).add(sp.server_id)
        if mode == "tablewise":
            for t, o in tab_owner.items():
                if len(o) != 1:
                    raise ConfigError(f"table-wise mode needs one owner per table (table {t})")
            self.feat_owner = [next(iter(tab_owner[t])) for t in self.ftab]
            self.owned_feats = [[f for f in range(self.F) if self.feat_owner[f] == r] for r in range(world)]
        self.ops = ops if ops is not None else FlexOps(self.metas, placement, seed, rank, self.ftab, self.fops,
                                                       batch_size, self.device)
        from .pooling import op_code
        self.bag_ops = torch.tensor(np.repeat([op_code(o) for o in self.fops], batch_size).astype(np.int32),
                                    device=self.device)
        self.stats = ExchangeStats()
        self.profile = False
        self.timeline = []  # (phase, start_event, end_event) when profiling

    def _mark(self, phase):
        if not self.profile:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return (phase, ev)

    def _close(self, tok):
        if tok is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.timeline.append((tok[0], tok[1], ev))

    def phase_ms(self) -> dict:
        """[sync] summed device time per phase since the last call."""
        torch.cuda.synchronize()
        out = {}
        for ph, a, b in self.timeline:
            out[ph] = out.get(ph, 0.0) + a.elapsed_time(b)
        self.timeline = []
        return out

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        tok = self._mark("a2a")
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        self._close(tok)

    def lookup(self, indices: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor | None = None,
               check: bool = True) -> torch.Tensor:
        """Pool this rank's batch; returns out [B, F*D] f32 (sample-major)."""
        dev, B, F, D, W = self.device, self.B, self.F, self.D, self.world
        n_bags = B * F
        if out is None:
            out = torch.empty((B, F * D), dtype=torch.float32, device=dev)
        tok = self._mark("route")
        send_idx, dcount, bcount = self.ops.route_bucket(indices, offsets, W)
        self._close(tok)
        self.pooled_rows_last = 0
        # C1: counts, per-bag lengths, indices
        recv_cnt = torch.empty(W, dtype=torch.int64, device=dev)
        self._a2a(recv_cnt, dcount)
        send_h = dcount.cpu().tolist()
        recv_h = recv_cnt.cpu().tolist()
        recv_len = torch.empty((W, n_bags), dtype=torch.int32, device=dev)
        self._a2a(recv_len.view(-1), bcount.reshape(-1))
        recv_idx = torch.empty(max(sum(recv_h), 1), dtype=torch.int32, device=dev)
        self._a2a(recv_idx[:sum(recv_h)], send_idx, recv_h, send_h)
        self.stats.c1_bytes_sent += int(send_idx.numel()) * 4 + W * n_bags * 4 + W * 8
        self.stats.calls += 1
        base = np.concatenate([[0], np.cumsum(recv_h)]).astype(np.int64)
        if self.mode == "tablewise":
            mine = self.owned_feats[self.rank]
            rows = len(mine) * B
            pooled = torch.empty((W, max(rows, 1), D), dtype=torch.float32, device=dev)
            tok = self._mark("pool")
            for q in range(W):
                if rows:
                    lens = recv_len[q].view(F, B)[mine].reshape(-1)
                    self.ops.owner_pool(recv_idx[base[q]:], lens, mine, pooled[q, :rows], partial=False)
            self._close(tok)
            back = [len(self.owned_feats[r]) * B for r in range(W)]
            recv_pool = torch.empty((max(sum(back), 1), D), dtype=torch.float32, device=dev)
            send = pooled[:, :rows].reshape(W * rows, D) if rows else pooled.new_empty((0, D))
            self._a2a(recv_pool[:sum(back)], send, back, [rows] * W)
            self.stats.c2_bytes_sent += W * rows * D * 4
            o3 = out.view(B, F, D)
            r0 = 0
            for r in range(W):
                fs = self.owned_feats[r]
                if fs:
                    o3[:, fs, :] = recv_pool[r0:r0 + len(fs) * B].view(len(fs), B, D).transpose(0, 1)
                r0 += len(fs) * B
        else:
            part = torch.zeros((W, n_bags, D), dtype=torch.float64, device=dev)
            cnts = torch.zeros((W, n_bags), dtype=torch.int32, device=dev)
            allf = list(range(F))
            tok = self._mark("pool")
            for q in range(W):
                self.ops.owner_pool(recv_idx[base[q]:], recv_len[q], allf, part[q], partial=True, counts=cnts[q])
            self._close(tok)
            recv_part = torch.empty_like(part)
            recv_cnts = torch.empty_like(cnts)
            self._a2a(recv_part.view(-1), part.view(-1))
            self._a2a(recv_cnts.view(-1), cnts.view(-1))
            self.stats.c2_bytes_sent += part.numel() * 8 + cnts.numel() * 4
            tmp = torch.empty((n_bags, D), dtype=torch.float32, device=dev)
            self.ops.combine(recv_part, recv_cnts, self.bag_ops, tmp)
            out.view(B, F, D).copy_(tmp.view(F, B, D).transpose(0, 1))
        if check:
            self.ops.check((indices, offsets))
        return out


# ---------------------------------------------------------------------------------------
# Fused exchange over NVLink peer memory (no NCCL on the data path)
# ---------------------------------------------------------------------------------------

def _ptr(t):
    return None if t is None else t.data_ptr()


def _cai_tensor(ptr: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    """Zero-copy torch view of a raw device allocation (__cuda_array_interface__)."""
    typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8"}[dtype]

    class _Arr:
        pass
    a = _Arr()
    a.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                  "version": 3, "strides": None}
    return torch.as_tensor(a, device=device)


class DevBuffer:
    """cudaMalloc'd (IPC-exportable) buffer owned by libflexemb."""

    def __init__(self, nbytes: int):
        from . import _lib
        self._lib = _lib
        p = ctypes.c_void_p()
        _lib.check(_lib.lib.fx_dev_alloc(max(int(nbytes), 1), ctypes.byref(p)), "dev alloc")
        self.ptr = int(p.value)
        self.nbytes = int(nbytes)

    def handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        self._lib.check(self._lib.lib.fx_ipc_export(self.ptr, buf), "ipc export")
        return buf.raw

    def __del__(self):
        try:
            self._lib.lib.fx_dev_free(self.ptr)
        except Exception:
            pass


def _ipc_open(handle: bytes) -> int:
    from . import _lib
    p = ctypes.c_void_p()
    _lib.check(_lib.lib.fx_ipc_open(handle, ctypes.byref(p)), "ipc open")
    return int(p.value)


class PeerComm:
    """fx_comm (include/flexemb.h, SURVEY §8(b) fx_comm_init / fx_alltoallv):
    a byte all-to-allv over CUDA-IPC-mapped peer memory of one node, no NCCL.
    Collective constructor (handles are exchanged with torch.distributed)."""

    def __init__(self, slot_bytes: int, group=None):
        import torch.distributed as dist
        from . import _lib
        self._lib = _lib
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.slot_bytes = (int(slot_bytes) + 15) // 16 * 16
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.fx_comm_init(ctypes.byref(h), self.rank, self.world, self.slot_bytes), "comm init")
        self._h = h.value
        buf = ctypes.create_string_buffer(64)
        _lib.check(_lib.lib.fx_comm_handle(self._h, buf), "comm handle")
        handles = [None] * self.world
        dist.all_gather_object(handles, buf.raw, group=group)
        _lib.check(_lib.lib.fx_comm_connect(self._h, b"".join(handles)), "comm connect")

    def alltoallv(self, send: torch.Tensor, counts: torch.Tensor, displs: torch.Tensor, stream=None):
        """send: uint8 CUDA tensor; counts / displs: int64 CUDA [world] (bytes
        for each destination). Returns (recv [world, slot_bytes] uint8 copy,
        recv_counts int64 [world]): row s holds recv_counts[s] bytes from rank s."""
        L = self._lib
        L.check(L.lib.fx_alltoallv(self._h, send.data_ptr(), counts.data_ptr(), displs.data_ptr(),
                                   L.stream_ptr(stream)), "alltoallv")
        recv = torch.empty((self.world, self.slot_bytes), dtype=torch.uint8, device=send.device)
        rc = torch.empty(self.world, dtype=torch.int64, device=send.device)
        L.check(L.lib.fx_memcpy_async(recv.data_ptr(), L.lib.fx_comm_recv_buffer(self._h), recv.numel(),
                                      L.stream_ptr(stream)), "alltoallv recv")
        L.check(L.lib.fx_memcpy_async(rc.data_ptr(), L.lib.fx_comm_recv_counts(self._h), 8 * self.world,
                                      L.stream_ptr(stream)), "alltoallv counts")
        return recv, rc

    def status(self) -> tuple:
        """[sync] (slot overflow, barrier timeout) flags."""
        a, b = ctypes.c_int32(), ctypes.c_int32()
        self._lib.check(self._lib.lib.fx_comm_status(self._h, ctypes.byref(a), ctypes.byref(b)), "comm status")
        return a.value, b.value

    def __del__(self):
        try:
            self._lib.lib.fx_comm_destroy(self._h)
        except Exception:
            pass


class P2PShardedLookup:
    """Sharded lookup whose exchange rides on the gather+pool kernel itself.

    Per step (one process per GPU):
      requester: stage its CSR batch in an IPC-exported buffer (row-wise: K1
                 route + fx_bucket first, so each owner's slice is a CSR of
                 its own rows);
      barrier A: every rank's batch is staged;
      owner:     ONE K4 launch over all requesters' bags of the tables it
                 hosts: indices/offsets are read through IPC-mapped pointers
                 over NVLink, rows are gathered from local HBM, and the pooled
                 rows are stored straight into the requester's output (table-
                 wise: final f32 rows; row-wise: f64 partials into the
                 requester's per-source slot), with a system-scope fence;
      barrier B: all owners' stores have landed;
      requester: row-wise only -> K5 combine (ascending source rank).
    The pooled "all-to-all" therefore overlaps the HBM gather bag by bag."""

    def __init__(self, metas, placement, seed: int, feature_tables, feature_ops, batch_size: int, rank: int,
                 world: int, device, group=None, mode: str = "tablewise", max_nnz: int | None = None,
                 replicated_tables=(), partial_dtype: str = "f64", pushdown_threshold: int | None = None,
                 balance_replicated: bool = True):
        """`replicated_tables` (table-wise mode): tables held in full by every
        rank and pooled locally for the rank's own batch (no exchange); they
        must not appear in `placement`. The other tables are table-sharded.

        `pushdown_threshold` (row-wise mode): the reference's hierarchical
        plan (pooling.py:88-100, ranker.py:263-301). A (bag, rank) group of at
        least `threshold` indices is pushed down to its owner (one partial);
        a smaller group is raw-fetched: the requester's K5 reads its rows
        straight from the owner's shard over NVLink (peer loads through
        IPC-mapped shard memory, the analogue of the reference's RDMA READ)
        and combines them after the partials in position order, as
        combine_partials does (pooling.py:103-123). Per-bag counters
        (pushdown_groups, pushdown_rows, raw_rows) come with every result
        (`counters()`). None pushes every group down."""
        from . import _lib
        from .pooling import op_code
        from .store import table_block_device
        self._lib = _lib
        self.replicated = set(replicated_tables)
        big = [m.table_id for m in (metas.values() if isinstance(metas, dict) else metas) if m.num_rows > 2**31 - 1]
        if big:
            # the pushes stage row indices as int32 for the owners' K4
            raise ConfigError(f"tables {big} have more than 2^31-1 rows: the fused exchange stages int32 row ids")
        if partial_dtype not in ("f64", "f32"):
            raise ConfigError("partial_dtype must be 'f64' or 'f32'")
        # row-wise partials: f64 (bit-exact vs flat) or f32 (PartialResult semantics of the
        # reference, pooling.py:35-47 / combine_partials double rounding; half the NVLink bytes)
        self.pesz = 8 if partial_dtype == "f64" else 4
        if self.replicated and mode != "tablewise":
            raise ConfigError("replicated tables are supported in table-wise mode only")
        self.threshold = pushdown_threshold
        if pushdown_threshold is not None:
            if pushdown_threshold < 2:
                raise ConfigError(f"pushdown threshold must be >= 2, got {pushdown_threshold}")
        if mode not in ("tablewise", "rowwise"):
            raise ConfigError(f"unknown sharding mode {mode!r}")
        self.metas = {m.table_id: m for m in metas}
        self.rank, self.world, self.mode, self.group = rank, world, mode, group
        self.device = torch.device(device)
        self.B = batch_size
        self.ftab, self.fops = tuple(feature_tables), tuple(feature_ops)
        self.F = len(self.ftab)
        dims = {self.metas[t].dim for t in self.ftab}
        if len(dims) != 1:
            raise ConfigError("sharded lookup needs one embedding dim across features")
        self.D = D = dims.pop()
        B, F, W = self.B, self.F, world
        self.n_bags = n_bags = B * F
        self.ops = FlexOps(self.metas, placement, seed, rank, self.ftab, self.fops, B, self.device,
                           ipc_shards=pushdown_threshold is not None and mode == "rowwise")
        for t in self.replicated:
            if any(sp.table_id == t for sp in placement):
                raise ConfigError(f"replicated table {t} must not be in the sharded placement")
            self.ops.local[t] = (table_block_device(seed, t, self.metas[t].dim, 0, self.metas[t].num_rows,
                                                    device=self.device), 0, self.metas[t].num_rows)
        tab_owner = {}
        for sp in placement:
            tab_owner.setdefault(sp.table_id, set()).add(sp.server_id)
        if mode == "tablewise":
            for t, o in tab_owner.items():
                if len(o) != 1:
                    raise ConfigError(f"table-wise mode needs one owner per table (table {t})")
            self.tw_owner = [(-1 if t in self.replicated else next(iter(tab_owner[t]))) for t in self.ftab]
            # executor of every (requester, feature): the owner for sharded tables;
            # replicated tables can be pooled by ANY rank, so they are spread to
            # even out the per-rank gather work (deterministic: same on every rank)
            self.execu = self._assign_executors(W, balance_replicated)
            self.feat_owner = list(self.execu[rank])
        self.max_nnz = int(max_nnz) if max_nnz is not None else n_bags * 64
        # every rank must use the same slot geometry (requesters address peers' slots)
        agreed = [None] * W
        dist.all_gather_object(agreed, self.max_nnz, group=group)
        self.max_nnz = max(agreed)
        dev = self.device
        # IPC-exported staging buffers, two sets (pipelined mode alternates them)
        self.b_flags = DevBuffer(W * 8)
        if mode == "tablewise":
            # owner-side staging: one slot per requester holding the indices and
            # rebased offsets of the features this rank owns (pushed by requesters)
            # slot (q -> d): the features requester q has executed by rank d
            self.slot_feats = lambda q, d: [f for f in range(F) if self.execu[q][f] == d]
            self.slot_stride = [max(len(self.slot_feats(q, d)) for q in range(W)) for d in range(W)]
            offs_slot = lambda d: (self.slot_stride[d] * B + 1) * 8
            out_set = n_bags * D * 4
        else:
            offs_slot = lambda d: (n_bags + 1) * 8
            out_set = W * n_bags * D * self.pesz
        self.idx_set = W * self.max_nnz * 4               # bytes per set, uniform across ranks
        self.offs_set = [W * offs_slot(d) for d in range(W)]
        self.out_set = out_set
        self.b_idx = DevBuffer(2 * self.idx_set)
        self.b_offs = DevBuffer(2 * self.offs_set[rank])
        self.b_out = DevBuffer(2 * self.out_set)
        self.t_flags = _cai_tensor(self.b_flags.ptr, (W,), torch.int64, dev)
        self.t_flags.zero_()
        if mode == "tablewise":
            self.t_out = [_cai_tensor(self.b_out.ptr + p * out_set, (B, F * D), torch.float32, dev) for p in (0, 1)]
            if pushdown_threshold is not None:
                self.t_counters = [torch.zeros((3, n_bags), dtype=torch.int32, device=dev) for _ in (0, 1)]
        else:
            pdt = torch.float64 if self.pesz == 8 else torch.float32
            self.t_out = [_cai_tensor(self.b_out.ptr + p * out_set, (W, n_bags, D), pdt, dev) for p in (0, 1)]
            self.t_counts = [torch.zeros(W * n_bags + 1, dtype=torch.int32, device=dev) for _ in (0, 1)]
            self.t_scan = [torch.zeros(W * n_bags + 1, dtype=torch.int64, device=dev) for _ in (0, 1)]
            need = ctypes.c_size_t(0)
            if pushdown_threshold is None:
                _lib.check(_lib.lib.fx_rw_push(None, None, None, None, None, 0, None, n_bags, W, None, None, None,
                                               None, None, ctypes.byref(need), None), "rw push ws")
            else:
                _lib.check(_lib.lib.fx_rw_push_planned(None, None, None, None, None, None, 0, None, n_bags, W,
                                                       int(pushdown_threshold), None, None, None, None, None, 0,
                                                       None, None, None, None, None, 0, None, ctypes.byref(need),
                                                       None), "rw push ws")
                self.t_raw_off = [torch.zeros(n_bags + 1, dtype=torch.int64, device=dev) for _ in (0, 1)]
                self.t_raw_ptr = [torch.zeros(max(self.max_nnz, 1), dtype=torch.int64, device=dev) for _ in (0, 1)]
                self.t_counters = [torch.zeros((3, n_bags), dtype=torch.int32, device=dev) for _ in (0, 1)]
            self.t_ws = [torch.empty(max(need.value, 1), dtype=torch.uint8, device=dev) for _ in (0, 1)]
        torch.cuda.synchronize(dev)
        mine = [self.b_idx.handle(), self.b_offs.handle(), self.b_out.handle(), self.b_flags.handle()]
        allh = [None] * W
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        ptrs = []
        for q in range(W):
            if q == rank:
                ptrs.append((self.b_idx.ptr, self.b_offs.ptr, self.b_out.ptr, self.b_flags.ptr))
            else:
                opened = tuple(_ipc_open(h) for h in allh[q])
                self._opened.extend(opened)
                ptrs.append(opened)
        self.peer_ptrs = ptrs
        self.t_peer_flags = torch.tensor([p[3] for p in ptrs], dtype=torch.int64, device=dev)
        if pushdown_threshold is not None and mode == "rowwise":
            # every shard's base address as seen from this rank (raw fetch targets)
            mine_sh = {t: buf.handle() for t, buf in self.ops.shard_bufs.items()}
            all_sh = [None] * W
            dist.all_gather_object(all_sh, mine_sh, group=group)
            bases = []
            for sp in self.ops.shard_list:
                if sp.server_id == rank:
                    bases.append(self.ops.local[sp.table_id][0].data_ptr())
                else:
                    p_ = _ipc_open(all_sh[sp.server_id][sp.table_id])
                    self._opened.append(p_)
                    bases.append(p_)
            self.t_shard_base = torch.tensor(bases, dtype=torch.int64, device=dev)
        self.t_timeout = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = 0
        from .store import make_segments
        self.segs, self.t_dst_idx, self.t_dst_offs = [], [], []
        for p in (0, 1):
            # push targets: this requester's slot (set p) in every owner's staging
            self.t_dst_idx.append(torch.tensor([ptrs[d][0] + p * self.idx_set + rank * self.max_nnz * 4
                                                for d in range(W)], dtype=torch.int64, device=dev))
            self.t_dst_offs.append(torch.tensor([ptrs[d][1] + p * self.offs_set[d] + rank * offs_slot(d)
                                                 for d in range(W)], dtype=torch.int64, device=dev))
            # owner segments over every requester's bags (virtual bag space), set p
            segs = []
            vb = 0
            # requesters in the order rank+1, rank+2, ..., rank: the persistent
            # K4 warps walk the virtual bags in order, so at any moment each
            # owner stores into a different requester (a shifted all-to-all:
            # no GPU's NVLink ingress takes every owner's stores at once)
            for qi in range(W):
                q = (rank + 1 + qi) % W
                qout = ptrs[q][2] + p * out_set
                lidx = self.b_idx.ptr + p * self.idx_set + q * self.max_nnz * 4
                loffs = self.b_offs.ptr + p * self.offs_set[rank] + q * offs_slot(rank)
                if mode == "tablewise":
                    for j, f in enumerate(self.slot_feats(q, rank)):
                        data, rb, re = self.ops.local[self.ftab[f]]
                        segs.append(_lib.FxSegment(data.data_ptr(), rb, re, vb, vb + B, qout + f * D * 4, F * D, D,
                                                   D, op_code(self.fops[f]), lidx, loffs + j * B * 8))
                        vb += B
                else:
                    for f in range(F):
                        t = self.ftab[f]
                        if t in self.ops.local:
                            data, rb, re = self.ops.local[t]
                            tp = data.data_ptr()
                        else:
                            tp, rb, re = 0, 0, 0
                        segs.append(_lib.FxSegment(tp, rb, re, vb, vb + B,
                                                   qout + (rank * n_bags + f * B) * D * self.pesz, D, D, D,
                                                   op_code(self.fops[f]), lidx, loffs + f * B * 8))
                        vb += B
            self.n_vbags = vb
            self.n_segs = len(segs)
            self.segs.append(make_segments(segs, dev) if segs else None)
        if mode == "tablewise":
            pos = [0] * F
            for d in range(W):
                for j, f in enumerate(self.slot_feats(rank, d)):
                    pos[f] = j
            self.t_feat_owner = torch.tensor(self.feat_owner, dtype=torch.int32, device=dev)
            self.t_feat_pos = torch.tensor(pos, dtype=torch.int32, device=dev)
            self.t_feat_nrows = torch.tensor([self.metas[t].num_rows for t in self.ftab],
                                             dtype=torch.int64, device=dev)
        self.bag_ops = torch.tensor(np.repeat([op_code(o) for o in self.fops], B).astype(np.int32), device=dev)
        if mode == "rowwise":
            self._pp = [torch.tensor([self.b_out.ptr + p * out_set + s * n_bags * D * self.pesz for s in range(W)],
                                     dtype=torch.int64, device=dev) for p in (0, 1)]
            self._cptr = [torch.tensor([self.t_counts[p].data_ptr() + s * n_bags * 4 for s in range(W)],
                                       dtype=torch.int64, device=dev) for p in (0, 1)]
            self._tmp = [torch.empty((n_bags, D), dtype=torch.float32, device=dev) for _ in (0, 1)]
        self.profile = False
        self.timeline = []
        self.launches = 0  # our kernels launched (libflexemb), for bench accounting
        self._barrier_waits = []

    def _assign_executors(self, W: int, balance: bool):
        """[q][f] -> rank that pools requester q's bags of feature f. Sharded
        features go to their owner (W units of B bags each); a requester's
        replicated features stay local while its rank is under the mean load
        ceil(total / W), the rest go to the least-loaded rank."""
        F = self.F
        execu = [[self.tw_owner[f] if self.tw_owner[f] >= 0 else q for f in range(F)] for q in range(W)]
        repl = [f for f in range(F) if self.tw_owner[f] < 0]
        if not balance or not repl:
            return execu
        load = [0] * W
        for f in range(F):
            if self.tw_owner[f] >= 0:
                load[self.tw_owner[f]] += W
        cap = -(-(sum(load) + len(repl) * W) // W)
        for q in range(W):
            for f in repl:
                d = q if load[q] < cap else min(range(W), key=lambda r: (load[r], r != q, r))
                execu[q][f] = d
                load[d] += 1
        self.exec_load = load
        return execu

    def _barrier(self):
        self.launches += 1
        L = self._lib
        for ev in self._barrier_waits:  # consumers of the output set the next step reuses
            torch.cuda.current_stream(self.device).wait_event(ev)
        self._barrier_waits = []
        self.epoch += 1
        L.check(L.lib.fx_peer_barrier(self.b_flags.ptr, self.t_peer_flags.data_ptr(), self.rank, self.world,
                                      self.epoch, self.t_timeout.data_ptr(), L.stream_ptr()), "peer barrier")

    def _mark(self, phase):
        if not self.profile:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return (phase, ev)

    def _close(self, tok):
        if tok is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.timeline.append((tok[0], tok[1], ev))

    def phase_ms(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for ph, a, b in self.timeline:
            out[ph] = out.get(ph, 0.0) + a.elapsed_time(b)
        self.timeline = []
        return out

    def _stage(self, indices, offsets, p, stream=None, hit_slot=None, cache_rows=0, cache_ld=0):
        """Ingress validation + push of this rank's batch into every owner's
        staging (set p). Row-wise planned mode: occurrences with
        hit_slot >= 0 are served from the requester's cache rows."""
        L = self._lib
        B, F, W = self.B, self.F, self.world
        nnz = int(indices.numel())
        self._last_batch = (indices, offsets)
        if nnz > self.max_nnz:
            raise ConfigError(f"batch has {nnz} indices, staging holds {self.max_nnz}")
        o = self.ops
        sp = L.stream_ptr(stream)
        # The table-wise push can validate while it copies (FX_PUSH_VALIDATE=1),
        # but measured slower: the short fused push runs in a burst against the
        # start of the concurrent gather, while the separate K1 pass spreads the
        # push across it (N=2 cfg2, same box: 1,126 vs 1,213 M bags/s;
        # scripts/run_stage_ab.sh, profiles/r1_summary.md).
        fused_validate = self.mode == "tablewise" and os.environ.get("FX_PUSH_VALIDATE", "0") == "1"
        if not fused_validate:
            L.check(L.lib.fx_route(o.route_off.data_ptr(), o.starts.data_ptr(), o.owners.data_ptr(),
                                   o.nrows.data_ptr(), o.bag_table.data_ptr(), indices.data_ptr(),
                                   L.idx_type_of(indices), offsets.data_ptr(), self.n_bags, None,
                                   o.status.err.data_ptr(), o.status.code.data_ptr(), sp), "validate")
        if self.mode == "tablewise":
            if self.threshold is not None:
                # a table-wise bag is ONE (bag, owner) group of L rows: pushed down
                # when L >= threshold, otherwise its rows are raw (ranker.py:281-293).
                # A raw group's pooled value is its row sum, which the owner's K4
                # produces bit-identically, so only the counters follow the plan.
                lens = (offsets[1:] - offsets[:-1]).to(torch.int32)
                push = lens >= int(self.threshold)
                c = self.t_counters[p]
                c[0].copy_(push.to(torch.int32))
                c[1].copy_(torch.where(push, lens, torch.zeros_like(lens)))
                c[2].copy_(torch.where(push, torch.zeros_like(lens), lens))
            self.launches += 1 if fused_validate else 2  # [k_route (validate)] + k_push_csr
            L.check(L.lib.fx_push_csr(indices.data_ptr(), L.idx_type_of(indices), offsets.data_ptr(), B, F,
                                      self.t_feat_owner.data_ptr(), self.t_feat_pos.data_ptr(),
                                      self.t_dst_idx[p].data_ptr(), self.t_dst_offs[p].data_ptr(),
                                      self.t_feat_nrows.data_ptr() if fused_validate else None, o.status.err.data_ptr(),
                                      o.status.code.data_ptr(), 1, sp), "push")
        elif self.threshold is not None:
            wsb = ctypes.c_size_t(self.t_ws[p].numel())
            L.check(L.lib.fx_rw_push_planned(o.route_off.data_ptr(), o.starts.data_ptr(), o.owners.data_ptr(),
                                             o.nrows.data_ptr(), o.bag_table.data_ptr(), indices.data_ptr(),
                                             L.idx_type_of(indices), offsets.data_ptr(), self.n_bags, W,
                                             int(self.threshold), self.t_counts[p].data_ptr(),
                                             self.t_scan[p].data_ptr(), self.t_dst_idx[p].data_ptr(),
                                             self.t_dst_offs[p].data_ptr(), self.t_shard_base.data_ptr(), self.D,
                                             self.t_raw_off[p].data_ptr(), self.t_raw_ptr[p].data_ptr(),
                                             self.t_counters[p].data_ptr(), _ptr(hit_slot), cache_rows, cache_ld,
                                             self.t_ws[p].data_ptr(), ctypes.byref(wsb), sp), "rw push planned")
            # k_route, k_rw_count, k_rw_plan, k_rw_raw, k_rw_push_planned, k_rw_push_offsets
            self.launches += 6
        else:
            wsb = ctypes.c_size_t(self.t_ws[p].numel())
            L.check(L.lib.fx_rw_push(o.route_off.data_ptr(), o.starts.data_ptr(), o.owners.data_ptr(),
                                     o.bag_table.data_ptr(), indices.data_ptr(), L.idx_type_of(indices),
                                     offsets.data_ptr(), self.n_bags, W, self.t_counts[p].data_ptr(),
                                     self.t_scan[p].data_ptr(), self.t_dst_idx[p].data_ptr(),
                                     self.t_dst_offs[p].data_ptr(), self.t_ws[p].data_ptr(), ctypes.byref(wsb), sp),
                    "rw push")
            self.launches += 4  # k_route (validate), k_rw_count, k_rw_push, k_rw_push_offsets

    def _gather(self, p):
        """ONE K4 launch over every requester's bags of this rank's tables,
        pooled rows stored into the requesters' output buffers (set p)."""
        L = self._lib
        if not self.n_segs:
            return
        self.launches += 1
        mode = (L.FX_OUT_F32 if self.mode == "tablewise" else
                (L.FX_OUT_F64_PARTIAL if self.pesz == 8 else L.FX_OUT_F32_PARTIAL))
        L.check(L.lib.fx_gather_pool(self.segs[p].data_ptr(), self.n_segs, self.D, self.b_idx.ptr, L.FX_IDX_I32,
                                     None, self.n_vbags, mode | L.FX_OUT_SYSFENCE, None,
                                     self.ops.owner_status.err.data_ptr(), L.FX_E_ROUTING_VIOLATION,
                                     self.ops.owner_status.code.data_ptr(), L.stream_ptr()), "fused pool")

    def _result(self, p, sample_major: bool = True):
        """Pooled [B, F*D] f32 of the step that used set p (row-wise: K5 first,
        writing sample-major rows directly; table-major [F*B, D] when
        sample_major is False)."""
        if self.mode == "tablewise":
            self._last_set = p
            return self.t_out[p]
        L = self._lib
        B, F, D, W = self.B, self.F, self.D, self.world
        self.launches += 1
        self._last_set = p
        planned = self.threshold is not None
        L.check(L.lib.fx_combine_ptr(self._pp[p].data_ptr(), 1 if self.pesz == 4 else 0, self._cptr[p].data_ptr(),
                                     W, D, self.t_raw_off[p].data_ptr() if planned else None,
                                     self.t_raw_ptr[p].data_ptr() if planned else None, self.n_bags, D, 0,
                                     self.bag_ops.data_ptr(), self._tmp[p].data_ptr(),
                                     F * D if sample_major else D, None, B if sample_major else 0,
                                     L.stream_ptr()), "combine")
        return self._tmp[p].view(B, F * D) if sample_major else self._tmp[p]

    def counters(self) -> torch.Tensor:
        """Per-bag (pushdown_groups, pushdown_rows, raw_rows) of the last result,
        int32 [3, F*B] in table-major bag order (ranker.py:281-293; needs a
        pushdown threshold)."""
        if self.threshold is None:
            raise ConfigError("counters need pushdown_threshold")
        return self.t_counters[self._last_set]

    def _check(self):
        self.ops.check(getattr(self, "_last_batch", None))
        if int(self.t_timeout.item()):
            raise RuntimeError("peer barrier timed out (a rank stopped participating)")

    def lookup(self, indices: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor | None = None,
               check: bool = True) -> torch.Tensor:
        """Pool this rank's batch synchronously (stage -> barrier -> fused
        gather -> barrier). Returns [B, F*D] f32 (the internal output buffer
        unless `out` is given; valid until the next call)."""
        tok = self._mark("stage")
        self._stage(indices, offsets, 0)
        self._close(tok)
        tok = self._mark("barrier")
        self._barrier()
        self._close(tok)
        tok = self._mark("pool")
        self._gather(0)
        self._close(tok)
        tok = self._mark("barrier")
        self._barrier()
        self._close(tok)
        tok = self._mark("combine")
        res = self._result(0)
        self._close(tok)
        if out is not None:
            out.copy_(res)
            res = out
        if check:
            self._check()
        return res

    def stream(self, batches, check: bool = True):
        """Pipelined lookups (the reference's pipeline_depth = 2): yields the
        pooled [B, F*D] of every (indices, offsets) batch, in order, one step
        behind submission. The push of step k+1 runs on a side stream while
        step k's fused gather runs, staging / outputs alternate between two
        buffer sets, and ONE barrier per step certifies both "every rank's push
        of step k landed" and "every rank's gather of step k-1 is done". A
        yielded tensor is valid until the generator is advanced again (in
        table-wise mode peer owners store the next-but-one step's rows into the
        same buffer as soon as the next barrier completes); consume or copy it
        on the current stream before advancing."""
        main = torch.cuda.current_stream(self.device)
        side = torch.cuda.Stream(self.device)
        # the gather runs on a high-priority stream so its blocks are scheduled
        # ahead of the concurrent push (same program order via stream waits)
        hp = torch.cuda.Stream(self.device, priority=-1) if os.environ.get("FX_GATHER_PRIORITY", "1") == "1" else None
        ev_bar = None
        k = 0
        for item in batches:
            indices, offsets = item[0], item[1]
            p = k % 2
            with torch.cuda.stream(side):
                if len(item) > 2 and item[2] is not None:
                    side.wait_event(item[2])  # the batch's inputs are ready (e.g. an H2D copy)
                if ev_bar is not None:
                    side.wait_event(ev_bar)  # set p free: gathers and combine of step k-2 done
                tok = self._mark("stage")
                self._stage(indices, offsets, p, stream=side)
                self._close(tok)
                ev_push = torch.cuda.Event()
                ev_push.record(side)
            main.wait_event(ev_push)
            tok = self._mark("barrier")
            self._barrier()
            self._close(tok)
            res = None
            if k >= 1:
                tok = self._mark("combine")
                res = self._result(1 - p)
                self._close(tok)
            # certifies for the restaging of set 1-p at step k+1: every owner's
            # gather of step k-1 is done (barrier k) and so is this rank's
            # combine of step k-1, which reads set 1-p's counts / raw lists
            ev_bar = torch.cuda.Event()
            ev_bar.record(main)
            if res is not None:
                yield res
            tok = self._mark("pool")
            if hp is not None:
                hp.wait_stream(main)
                with torch.cuda.stream(hp):
                    self._gather(p)
                main.wait_stream(hp)
            else:
                self._gather(p)
            self._close(tok)
            k += 1
        if k:
            tok = self._mark("barrier")
            self._barrier()
            self._close(tok)
            tok = self._mark("combine")
            res = self._result((k - 1) % 2)
            self._close(tok)
            yield res
        if check:
            self._check()

    def pool_cached(self, indices: torch.Tensor, offsets: torch.Tensor, hit_slot: torch.Tensor | None,
                    cache=None) -> torch.Tensor:
        """One synchronous step for a requester that has a cache (row-wise
        planned mode): occurrences with hit_slot >= 0 are combined from the
        cache's rows, the rest follow the plan (pushdown to the owner or raw
        fetch over NVLink). Returns the table-major pooled [F*B, D] f32."""
        if self.threshold is None or self.mode != "rowwise":
            raise ConfigError("pool_cached needs the planned row-wise mode (pushdown_threshold)")
        rows, ld = cache.rows_base() if (cache is not None and hit_slot is not None) else (0, 0)
        self._stage(indices, offsets, 0, hit_slot=hit_slot, cache_rows=rows, cache_ld=ld)
        self._barrier()
        self._gather(0)
        self._barrier()
        return self._result(0, sample_major=False)

    def stream_host(self, host_batches, check: bool = True):
        """End-to-end pipelined API: pinned host (indices, offsets) in, pinned
        host pooled [B, F*D] f32 out, one per batch, in order. H2D copies run
        on their own stream into 3 rotating device slots, the fused exchange
        runs as in `stream()`, and each result's D2H runs on a copy stream
        overlapping the next step's gather; the barrier that lets owners
        overwrite that output set waits for the copy. A yielded tensor is
        valid until the generator is advanced."""
        dev = self.device
        main = torch.cuda.current_stream(dev)
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        slots = [dict(idx=None, offs=None, ev=torch.cuda.Event(), used=None) for _ in range(3)]
        host = [torch.empty((self.B, self.F * self.D), dtype=torch.float32, pin_memory=True) for _ in range(2)]
        ev_d2h = [torch.cuda.Event() for _ in range(2)]
        consumed = {}

        def dev_iter():
            for j, (ih, oh) in enumerate(host_batches):
                sl = slots[j % 3]
                with torch.cuda.stream(s_h2d):
                    if j >= 3:
                        s_h2d.wait_event(consumed.pop(j - 3))  # step j-3's push has read the slot
                    if sl["idx"] is None or sl["idx"].numel() < ih.numel() or sl["idx"].dtype != ih.dtype:
                        sl["idx"] = torch.empty(max(int(ih.numel()), 1), dtype=ih.dtype, device=dev)
                        sl["offs"] = torch.empty(oh.numel(), dtype=torch.int64, device=dev)
                    di, do = sl["idx"][:ih.numel()], sl["offs"][:oh.numel()]
                    di.copy_(ih, non_blocking=True)
                    do.copy_(oh, non_blocking=True)
                    sl["ev"].record(s_h2d)
                yield di, do, sl["ev"]

        prev = None
        for i, res in enumerate(self.stream(dev_iter(), check=check)):
            ev = torch.cuda.Event()
            ev.record(main)  # pushes of steps <= i+1 are done by now in main's order
            consumed[i] = ev
            k = i % 2
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev)
                host[k].copy_(res, non_blocking=True)
                ev_d2h[k].record(s_d2h)
            self._barrier_waits.append(ev_d2h[k])
            if prev is not None:
                ev_d2h[prev].synchronize()
                yield host[prev]
            prev = k
        if prev is not None:
            ev_d2h[prev].synchronize()
            yield host[prev]

    def close(self):
        L = self._lib
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            L.lib.fx_ipc_close(p)
        self._opened = []
