"""Multi-GPU sharded lookup: one process per GPU, tables table-wise or
row-wise sharded in HBM across the ranks of one box, pooled results returned
to the requesting GPU over NCCL all-to-all (NVLink 5 / NVSwitch).

This replaces the reference's fan-out seam (ranker.py:263-347 _fan_out ->
VirtualTransport.post_subrequest -> _server_handler -> _on_response): a
"server" is a GPU rank, a subrequest is the slice of a requester's CSR batch
routed to that rank, and the response is pooled vectors (pushdown):

  requester: K1 fx_route (index -> owning rank) + fx_bucket (stable per-rank
             CSR, GroupItem.positions semantics)            routing.py:117-148
  C1:        all_to_all of per-bag lengths + indices
  owner:     K4 gather+pool over its local shards: table-wise -> final f32
             (whole bag local, one rounding); row-wise -> f64 partial + count
             (PartialResult(sum, count), store.py:184-193)
  C2:        all_to_all of pooled rows back to the requester
  requester: table-wise -> placement into out[B, F*D];
             row-wise -> K5 fx_combine in ascending source rank (pooling.py:103-123)

Every rank runs the same per-GPU batch shape (weak scaling). Works with any
torch.distributed backend (NCCL on GPUs; the CPU tests drive the host logic
with gloo).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError
from .pooling import op_code
from .store import ShardSpec, TableMeta, make_segments, table_block_device


def tablewise_placement(table_rows, world: int):
    """Greedy balance of tables over ranks by row count (largest first);
    one shard per table (cfg4 placement)."""
    order = sorted(range(len(table_rows)), key=lambda t: -table_rows[t])
    load = [0] * world
    owner = [0] * len(table_rows)
    for t in order:
        r = min(range(world), key=lambda i: (load[i], i))
        owner[t] = r
        load[r] += table_rows[t]
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


@dataclass
class ExchangeStats:
    c1_bytes_sent: int = 0
    c2_bytes_sent: int = 0


class ShardedLookup:
    """Per-rank sharded lookup engine.

    `feature_tables` fixes the batch layout (feature f reads table
    feature_tables[f]); every rank submits batches of `batch_size` samples,
    table-major CSR (bag = f*B + s)."""

    def __init__(self, metas, placement, seed: int, feature_tables, feature_ops, batch_size: int,
                 rank: int, world: int, device, group=None, mode: str = "tablewise"):
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
        # local shards
        self.local = {}  # table -> (tensor, start, end)
        for sp in placement:
            if sp.server_id == rank:
                if sp.table_id in self.local:
                    raise ConfigError("one shard per table per rank")
                data = table_block_device(seed, sp.table_id, self.metas[sp.table_id].dim, sp.start, sp.end,
                                          device=self.device)
                self.local[sp.table_id] = (data, sp.start, sp.end)
        # routing tables on device: per table sorted starts + owning rank
        n_t = max(self.metas) + 1
        route_off = np.zeros(n_t + 1, np.int64)
        starts, owners = [], []
        for t in range(n_t):
            sh = sorted((s for s in placement if s.table_id == t), key=lambda s: s.start)
            route_off[t + 1] = route_off[t] + len(sh)
            starts += [s.start for s in sh]
            owners += [s.server_id for s in sh]
        nrows = np.array([self.metas[t].num_rows if t in self.metas else 0 for t in range(n_t)], np.int64)
        dev = self.device
        self.route_off = torch.from_numpy(route_off).to(dev)
        self.starts = torch.tensor(starts, dtype=torch.int64, device=dev)
        self.owners = torch.tensor(owners, dtype=torch.int32, device=dev)
        self.nrows = torch.from_numpy(nrows).to(dev)
        self.bag_table = torch.tensor(np.repeat(np.array(self.ftab, np.int32), batch_size), device=dev)
        self.status = _lib.Status(dev)
        self.stats = ExchangeStats()
        # table-wise: which features each rank owns (whole tables)
        tab_owner = {}
        for sp in placement:
            tab_owner.setdefault(sp.table_id, set()).add(sp.server_id)
        if mode == "tablewise":
            for t, o in tab_owner.items():
                if len(o) != 1:
                    raise ConfigError(f"table-wise mode needs one owner per table (table {t})")
            self.feat_owner = [next(iter(tab_owner[t])) for t in self.ftab]
            self.owned_feats = [[f for f in range(self.F) if self.feat_owner[f] == r] for r in range(world)]
        n_bags = self.F * batch_size
        self._ws = None
        self._perm = torch.empty(1, dtype=torch.int64, device=dev)
        self._dcount = torch.empty(world, dtype=torch.int64, device=dev)
        self._bcount = torch.empty(world * n_bags, dtype=torch.int32, device=dev)
        self._seg_cache = {}

    # ---------------------------------------------------------------------------------

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def _owner_segments(self, out, n_rows_out_per_req, mode_partial, requester_feats):
        """Segments for the owner's K4 over one requester's bags."""
        key = (out.data_ptr(), mode_partial, tuple(requester_feats))
        if key in self._seg_cache:
            return self._seg_cache[key]
        B, D = self.B, self.D
        segs = []
        esz = 8 if mode_partial else 4
        for j, f in enumerate(requester_feats):
            t = self.ftab[f]
            if t in self.local:
                data, start, end = self.local[t]
                tp, rb, re = data.data_ptr(), start, end
            else:  # no local shard: every bag of this feature has zero rows here
                tp, rb, re = 0, 0, 0
            segs.append(_lib.FxSegment(tp, rb, re, j * B, (j + 1) * B, out.data_ptr() + j * B * D * esz, D, D, D,
                                       op_code(self.fops[f])))
        seg = make_segments(segs, self.device)
        self._seg_cache[key] = seg
        if len(self._seg_cache) > 64:
            self._seg_cache.pop(next(iter(self._seg_cache)))
        return seg

    def lookup(self, indices: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor | None = None,
               check: bool = True) -> torch.Tensor:
        """Pool this rank's batch; returns out [B, F*D] f32 (sample-major)."""
        dev, B, F, D, W = self.device, self.B, self.F, self.D, self.world
        n_bags = B * F
        nnz = int(indices.numel())
        if out is None:
            out = torch.empty((B, F * D), dtype=torch.float32, device=dev)
        idx64 = indices.to(torch.int64) if indices.dtype != torch.int64 else indices
        # K1: owner rank per occurrence (validates ingress)
        dest = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        _lib.check(_lib.lib.fx_route(self.route_off.data_ptr(), self.starts.data_ptr(), self.owners.data_ptr(),
                                     self.nrows.data_ptr(), self.bag_table.data_ptr(), idx64.data_ptr(),
                                     _lib.FX_IDX_I64, offsets.data_ptr(), n_bags, dest.data_ptr(),
                                     self.status.err.data_ptr(), self.status.code.data_ptr(), _lib.stream_ptr()),
                   "route")
        # stable bucket per destination rank
        need = ctypes.c_size_t(0)
        _lib.check(_lib.lib.fx_bucket(None, nnz, None, n_bags, W, None, None, None, None, ctypes.byref(need), None))
        if self._ws is None or self._ws.numel() < need.value:
            self._ws = torch.empty(max(need.value, 1), dtype=torch.uint8, device=dev)
        if self._perm.numel() < max(nnz, 1):
            self._perm = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        _lib.check(_lib.lib.fx_bucket(dest.data_ptr(), nnz, offsets.data_ptr(), n_bags, W, self._perm.data_ptr(),
                                      self._dcount.data_ptr(), self._bcount.data_ptr(), self._ws.data_ptr(),
                                      ctypes.byref(need), _lib.stream_ptr()), "bucket")
        send_idx = idx64[self._perm[:nnz]].to(torch.int32)
        # C1a: counts per destination (1 int64 each), C1b: per-bag lengths, C1c: indices
        recv_cnt = torch.empty(W, dtype=torch.int64, device=dev)
        self._a2a(recv_cnt, self._dcount)
        send_cnt_h = self._dcount.cpu().tolist()
        recv_cnt_h = recv_cnt.cpu().tolist()
        recv_len = torch.empty(W * n_bags, dtype=torch.int32, device=dev)
        self._a2a(recv_len, self._bcount)
        recv_idx = torch.empty(max(sum(recv_cnt_h), 1), dtype=torch.int32, device=dev)
        self._a2a(recv_idx[:sum(recv_cnt_h)], send_idx, recv_cnt_h, send_cnt_h)
        self.stats.c1_bytes_sent += (nnz * 4 + W * n_bags * 4 + W * 8)
        recv_len = recv_len.view(W, n_bags)
        # owner side: pool every requester's bags over the local shards
        if self.mode == "tablewise":
            mine = self.owned_feats[self.rank]
            rows_per_req = len(mine) * B
            pooled = torch.empty((W, max(rows_per_req, 1), D), dtype=torch.float32, device=dev)
            base = 0
            for q in range(W):
                lens_q = recv_len[q].view(F, B)[mine].reshape(-1) if mine else recv_len[q][:0]
                offs_q = torch.zeros(rows_per_req + 1, dtype=torch.int64, device=dev)
                offs_q[1:] = torch.cumsum(lens_q.long(), 0)
                if rows_per_req:
                    seg = self._owner_segments(pooled[q], B, False, mine)
                    _lib.check(_lib.lib.fx_gather_pool(seg.data_ptr(), len(mine), D, recv_idx[base:].data_ptr(),
                                                       _lib.FX_IDX_I32, offs_q.data_ptr(), rows_per_req,
                                                       _lib.FX_OUT_F32, None, self.status.err.data_ptr(),
                                                       _lib.FX_E_ROUTING_VIOLATION, self.status.code.data_ptr(),
                                                       _lib.stream_ptr()), "owner pool")
                base += recv_cnt_h[q]
            # C2: pooled rows back to requesters (sizes known a priori)
            back = [len(self.owned_feats[r]) * B for r in range(W)]
            recv_pool = torch.empty((sum(back), D), dtype=torch.float32, device=dev)
            self._a2a(recv_pool, pooled[:, :rows_per_req].reshape(W * rows_per_req, D) if rows_per_req
                      else pooled.new_empty((0, D)), [b for b in back], [rows_per_req] * W)
            self.stats.c2_bytes_sent += W * rows_per_req * D * 4
            # placement into out[B, F*D]
            o3 = out.view(B, F, D)
            r0 = 0
            for r in range(W):
                fs = self.owned_feats[r]
                if fs:
                    blk = recv_pool[r0:r0 + len(fs) * B].view(len(fs), B, D).transpose(0, 1)
                    o3[:, fs, :] = blk
                r0 += len(fs) * B
        else:
            # row-wise: f64 partial + count per (bag, source rank)
            part = torch.zeros((W, n_bags, D), dtype=torch.float64, device=dev)
            cnts = torch.zeros((W, n_bags), dtype=torch.int32, device=dev)
            base = 0
            allf = list(range(F))
            for q in range(W):
                offs_q = torch.zeros(n_bags + 1, dtype=torch.int64, device=dev)
                offs_q[1:] = torch.cumsum(recv_len[q].long(), 0)
                seg = self._owner_segments(part[q], B, True, allf)
                _lib.check(_lib.lib.fx_gather_pool(seg.data_ptr(), F, D, recv_idx[base:].data_ptr(),
                                                   _lib.FX_IDX_I32, offs_q.data_ptr(), n_bags,
                                                   _lib.FX_OUT_F64_PARTIAL, cnts[q].data_ptr(),
                                                   self.status.err.data_ptr(), _lib.FX_E_ROUTING_VIOLATION,
                                                   self.status.code.data_ptr(), _lib.stream_ptr()), "owner pool")
                base += recv_cnt_h[q]
            recv_part = torch.empty_like(part)
            recv_cnts = torch.empty_like(cnts)
            self._a2a(recv_part.view(-1), part.view(-1))
            self._a2a(recv_cnts.view(-1), cnts.view(-1))
            self.stats.c2_bytes_sent += part.numel() * 8 + cnts.numel() * 4
            # K5: fold partials in ascending source rank, write sample-major
            ptrs = torch.tensor([recv_part[s].data_ptr() for s in range(W)], dtype=torch.int64, device=dev)
            cptr = torch.tensor([recv_cnts[s].data_ptr() for s in range(W)], dtype=torch.int64, device=dev)
            ops = torch.tensor(np.repeat([op_code(o) for o in self.fops], B).astype(np.int32), device=dev)
            tmp = torch.empty((n_bags, D), dtype=torch.float32, device=dev)
            _lib.check(_lib.lib.fx_combine(ptrs.data_ptr(), cptr.data_ptr(), W, D, None, None, n_bags, D, 0,
                                           ops.data_ptr(), tmp.data_ptr(), D, None, _lib.stream_ptr()), "combine")
            out.view(B, F, D).copy_(tmp.view(F, B, D).transpose(0, 1))
        if check:
            code, pos = self.status.read()
            if code:
                self.status.reset()
                from .errors import LookupValidationError, RoutingViolationError
                exc = LookupValidationError if code == _lib.FX_E_LOOKUP_VALIDATION else RoutingViolationError
                raise exc(f"bad index at CSR position {pos} on rank {self.rank}")
        return out
