"""Batched single-GPU lookup engine: the hot path behind Ranker.execute_batch.

A batch is KJT-like CSR: `indices` [nnz] (int32/int64) and `offsets`
[n_bags+1] (int64) with bags TABLE-MAJOR (bag = f*B + s for feature slot f
and sample s), so each feature is one contiguous bag segment reading one
HBM-resident table. One fx_gather_pool (K4) launch pools every bag of the
batch, validates every index at ingress (bad index -> LookupValidationError,
ranker.py:184-193) and writes the pooled f32 vectors sample-major into
out[B, F*D] (out[s, f*D:(f+1)*D] = bag (s, f)).
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, LookupValidationError
from .pooling import op_code
from .store import make_segments


@dataclass
class CsrBatch:
    """Device (or pinned host) CSR batch, table-major bags."""

    indices: torch.Tensor
    offsets: torch.Tensor
    feature_tables: tuple
    feature_ops: tuple
    batch_size: int

    @property
    def n_features(self) -> int:
        return len(self.feature_tables)

    @property
    def n_bags(self) -> int:
        return self.offsets.numel() - 1

    def to(self, device, non_blocking=True) -> "CsrBatch":
        return CsrBatch(self.indices.to(device, non_blocking=non_blocking),
                        self.offsets.to(device, non_blocking=non_blocking),
                        self.feature_tables, self.feature_ops, self.batch_size)

    def pin_memory(self) -> "CsrBatch":
        return CsrBatch(self.indices.pin_memory(), self.offsets.pin_memory(), self.feature_tables,
                        self.feature_ops, self.batch_size)


class LookupEngine:
    """Pools CSR batches against the deployment's shards resident on one GPU.

    Every table must be a single shard hosted on this device (table-wise or
    single-GPU placement); multi-shard tables go through ShardedLookup."""

    def __init__(self, deployment, device=None):
        self.dep = deployment
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.tables: dict = {}
        for sid, server in deployment.servers.items():
            for t in server.hosted_tables():
                shards = server.shards(t)
                for sh in shards:
                    if sh.data is None:
                        continue
                    if sh.data.device != self.device:
                        continue
                    if sh.start != 0 or sh.end != deployment.meta(t).num_rows:
                        continue
                    self.tables[t] = sh.data
        self.status = _lib.Status(self.device)
        self._segs: OrderedDict = OrderedDict()
        self._seg_cap = 16  # cached segment descriptor sets (raised by capture)

    def dim_of(self, t: int) -> int:
        return self.dep.meta(t).dim

    def _segments(self, batch: CsrBatch, out: torch.Tensor) -> torch.Tensor:
        key = (batch.feature_tables, batch.feature_ops, batch.batch_size, out.data_ptr(), out.stride(0))
        seg = self._segs.get(key)
        if seg is not None:
            self._segs.move_to_end(key)
            return seg
        B = batch.batch_size
        segs = []
        col = 0
        for f, (t, op) in enumerate(zip(batch.feature_tables, batch.feature_ops)):
            if t not in self.tables:
                raise ConfigError(f"table {t} is not resident as one shard on {self.device}")
            tab = self.tables[t]
            D = tab.shape[1]
            segs.append(_lib.FxSegment(tab.data_ptr(), 0, tab.shape[0], f * B, (f + 1) * B,
                                       out.data_ptr() + col * 4, out.stride(0), tab.stride(0), D, op_code(op)))
            col += D
        seg = make_segments(segs, self.device)
        self._segs[key] = seg
        if len(self._segs) > self._seg_cap:
            self._segs.popitem(last=False)
        return seg

    def out_dim(self, batch: CsrBatch) -> int:
        return sum(self.dim_of(t) for t in batch.feature_tables)

    def pool(self, batch: CsrBatch, out: torch.Tensor | None = None, check: bool = True,
             stream=None, status=None) -> torch.Tensor:
        """Launch K4 for the whole batch; returns out [B, sum(D_f)] f32."""
        B = batch.batch_size
        if batch.n_bags != B * batch.n_features:
            raise ConfigError("offsets must describe batch_size * n_features table-major bags")
        if out is None:
            out = torch.empty((B, self.out_dim(batch)), dtype=torch.float32, device=self.device)
        _lib.check_out(out, B, self.out_dim(batch))
        dims = {self.dim_of(t) for t in batch.feature_tables}
        st_ = status or self.status
        if len(dims) != 1:
            return self._pool_mixed(batch, out, check, stream, st_)
        D = dims.pop()
        segs = self._segments(batch, out)
        aligned = _lib.vec_ok((out.data_ptr(), out.stride(0)), (D * 4, 0),
                              *[(self.tables[t].data_ptr(), self.tables[t].stride(0)) for t in batch.feature_tables])
        _lib.check(_lib.lib.fx_gather_pool(segs.data_ptr(), batch.n_features, D, batch.indices.data_ptr(),
                                           _lib.idx_type_of(batch.indices), batch.offsets.data_ptr(), batch.n_bags,
                                           _lib.FX_OUT_F32 | (0 if aligned else _lib.FX_OUT_SCALAR), None,
                                           st_.err.data_ptr(),
                                           _lib.FX_E_LOOKUP_VALIDATION, st_.code.data_ptr(),
                                           _lib.stream_ptr(stream)), "gather_pool")
        if check:
            self.raise_if_bad(batch)
        return out

    def _pool_mixed(self, batch, out, check, stream, status=None):
        status = status or self.status
        # one launch per distinct dim; segments of other dims are skipped by
        # giving the kernel only the bags of the matching features
        segs_all = []
        B = batch.batch_size
        col = 0
        for f, t in enumerate(batch.feature_tables):
            D = self.dim_of(t)
            segs_all.append((f, t, D, col))
            col += D
        for D in sorted({s[2] for s in segs_all}):
            for f, t, d, c in segs_all:
                if d != D:
                    continue
                tab = self.tables[t]
                seg = make_segments([_lib.FxSegment(tab.data_ptr(), 0, tab.shape[0], 0, B, out.data_ptr() + c * 4,
                                                    out.stride(0), tab.stride(0), D,
                                                    op_code(batch.feature_ops[f]))], self.device)
                offs = batch.offsets[f * B:(f + 1) * B + 1]
                # mixed dims: a feature's output column offset need not be 16-B aligned
                aligned = _lib.vec_ok((out.data_ptr() + c * 4, out.stride(0)), (tab.data_ptr(), tab.stride(0)))
                _lib.check(_lib.lib.fx_gather_pool(seg.data_ptr(), 1, D, batch.indices.data_ptr(),
                                                   _lib.idx_type_of(batch.indices), offs.data_ptr(), B,
                                                   _lib.FX_OUT_F32 | (0 if aligned else _lib.FX_OUT_SCALAR), None,
                                                   status.err.data_ptr(),
                                                   _lib.FX_E_LOOKUP_VALIDATION, status.code.data_ptr(),
                                                   _lib.stream_ptr(stream)), "gather_pool")
        if check:
            self.raise_if_bad(batch)
        return out

    def prepare_many(self, batches, outs=None) -> "ManyPlan":
        """Build (once) the segment descriptors for pooling several
        independent requests in ONE K4 launch (see pool_many); the returned
        plan relaunches with no host-side work beyond the launch itself, for
        serving loops whose request slots are reused."""
        if not batches:
            raise ConfigError("prepare_many: no requests")
        dims = {self.dim_of(t) for b in batches for t in b.feature_tables}
        if len(dims) != 1:
            raise ConfigError("pool_many needs one embedding dim across requests")
        D = dims.pop()
        if len({b.indices.dtype for b in batches}) != 1:
            raise ConfigError("pool_many needs one index dtype across requests")
        if outs is None:
            outs = [torch.empty((b.batch_size, self.out_dim(b)), dtype=torch.float32, device=self.device)
                    for b in batches]
        segs, vb = [], 0
        for b, o in zip(batches, outs):
            B = b.batch_size
            if b.n_bags != B * b.n_features:
                raise ConfigError("offsets must describe batch_size * n_features table-major bags")
            for f, (t, op) in enumerate(zip(b.feature_tables, b.feature_ops)):
                if t not in self.tables:
                    raise ConfigError(f"table {t} is not resident as one shard on {self.device}")
                tab = self.tables[t]
                segs.append(_lib.FxSegment(tab.data_ptr(), 0, tab.shape[0], vb, vb + B,
                                           o.data_ptr() + f * D * 4, o.stride(0), tab.stride(0), D, op_code(op),
                                           b.indices.data_ptr(), b.offsets.data_ptr() + f * B * 8))
                vb += B
        return ManyPlan(self, list(batches), outs, make_segments(segs, self.device), len(segs), vb, D)

    def pool_many(self, batches, outs=None, check: bool = True, stream=None):
        """Pool several independent requests (e.g. the concurrent request
        streams of SURVEY §8(d) cfg5, or small serving requests) in ONE K4
        launch: every (request, feature) is a segment carrying its own index
        and offset arrays (fx_segment.idx / .offs), laid out one after the
        other in a virtual bag space, so small requests share one grid instead
        of paying a launch each. Same arithmetic and bit-identical results as
        pool() per request. Returns the list of [B_r, sum D] outputs."""
        if not batches:
            return []
        plan = self.prepare_many(batches, outs)
        plan.launch(stream)
        if check:
            plan.check()
        return plan.outs

    def capture(self, batches, outs, stream=None):
        """Capture one K4 launch per (batch, out) pair into a CUDA graph
        (small batches are launch-bound: cfg1 moves ~21 MB per batch). The
        segment descriptors are uploaded before capture; replay with
        graph.replay(); check status with raise_if_bad() afterwards."""
        self._seg_cap = max(self._seg_cap, len(batches) + 16)  # every descriptor set stays resident
        for b, o in zip(batches, outs):
            self._segments(b, o)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        s = stream or torch.cuda.Stream(self.device)
        with torch.cuda.graph(g, stream=s):
            for b, o in zip(batches, outs):
                self.pool(b, out=o, check=False)
        return g

    def raise_if_bad(self, batch: CsrBatch, batch_id: int = 0) -> None:
        """[sync] Raise LookupValidationError for the first bad index in
        (lookup, feature, position) order, with the reference's message
        (ranker.py:184-193)."""
        code, pos = self.status.read()
        if not code:
            return
        self.status.reset()
        best = self._first_bad(batch)
        if best is None:
            raise LookupValidationError(f"batch {batch_id}: an index was out of range (batch changed since launch)")
        s, f, index, t, n = best
        raise LookupValidationError(f"batch {batch_id}, lookup {s}: index {index} out of range [0,{n}) for table {t}")

    def _first_bad(self, batch: CsrBatch):
        """First out-of-range index in (lookup, feature, position) order, or None."""
        offs = batch.offsets.cpu().numpy()
        idx = batch.indices.cpu().numpy()
        B = batch.batch_size
        best = None
        for f, t in enumerate(batch.feature_tables):
            n = self.dep.meta(t).num_rows
            for s in range(B):
                b = f * B + s
                seg = idx[offs[b]:offs[b + 1]]
                bad = np.nonzero((seg < 0) | (seg >= n))[0]
                if bad.size:
                    cand = (s, f, int(seg[bad[0]]), t, n)
                    if best is None or cand[:2] < best[:2]:
                        best = cand
        return best


def algorithmic_bytes(batch_nnz: int, n_bags: int, dim: int, idx_bytes: int = 4) -> int:
    """per bag L*D*4 (rows) + L*idx (indices) + 8 (offset) + D*4 (pooled write)."""
    return batch_nnz * dim * 4 + batch_nnz * idx_bytes + n_bags * 8 + n_bags * dim * 4


class ManyPlan:
    """Prepared multi-request K4 launch (LookupEngine.prepare_many)."""

    def __init__(self, eng, batches, outs, segs, n_segs, n_vbags, dim):
        self.eng, self.batches, self.outs = eng, batches, outs
        self.segs, self.n_segs, self.n_vbags, self.dim = segs, n_segs, n_vbags, dim
        self._idx_type = _lib.idx_type_of(batches[0].indices)
        self._idx0 = batches[0].indices.data_ptr()

    def launch(self, stream=None) -> None:
        e = self.eng
        _lib.check(_lib.lib.fx_gather_pool(self.segs.data_ptr(), self.n_segs, self.dim, self._idx0, self._idx_type,
                                           None, self.n_vbags, _lib.FX_OUT_F32, None, e.status.err.data_ptr(),
                                           _lib.FX_E_LOOKUP_VALIDATION, e.status.code.data_ptr(),
                                           _lib.stream_ptr(stream)), "gather_pool many")

    def check(self) -> None:
        """[sync] LookupValidationError naming the first request with a bad index."""
        e = self.eng
        code, _ = e.status.read()
        if not code:
            return
        e.status.reset()
        for r, b in enumerate(self.batches):
            best = e._first_bad(b)
            if best is not None:
                s, f, index, t, n = best
                raise LookupValidationError(f"request {r}, lookup {s}: index {index} out of range "
                                            f"[0,{n}) for table {t}")


class HostLookup:
    """Reference-facing host API over the engine: host (pinned) CSR in,
    host pooled [B, sum D] f32 out, synchronous like Ranker.execute_batch
    (validation errors raise after the call). Copies ride the engine stream."""

    def __init__(self, engine: LookupEngine):
        self.engine = engine
        self._out_host = {}
        self._streams = {}

    def _stream_state(self, depth: int) -> dict:
        st = self._streams.get(depth)
        if st is None:
            dev = self.engine.device
            st = {"streams": tuple(torch.cuda.Stream(dev) for _ in range(3)),
                  "slots": [{"idx": None, "offs": None, "out": None, "host": None, "used": False, "batch": None,
                             "ev_in": torch.cuda.Event(), "ev_cmp": torch.cuda.Event(),
                             "ev_out": torch.cuda.Event()} for _ in range(depth)]}
            self._streams[depth] = st
        return st

    def lookup(self, batch_host: CsrBatch, out_host: torch.Tensor | None = None) -> torch.Tensor:
        eng = self.engine
        dev_batch = batch_host.to(eng.device, non_blocking=True)
        out = eng.pool(dev_batch, check=False)
        if out_host is None:
            key = tuple(out.shape)
            out_host = self._out_host.get(key)
            if out_host is None:
                out_host = self._out_host[key] = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        out_host.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        eng.raise_if_bad(dev_batch)
        return out_host

    def stream(self, batches_host, depth: int = 3):
        """Pipelined host API (the reference's pipeline_depth batches in
        flight, ranker.py:161-168): yields one pinned host output per input
        batch, in order. H2D of batch i+1, K4 of batch i and D2H of batch i-1
        run concurrently on three streams (PCIe is full duplex), so steady
        state is bound by the larger copy, not by their sum. Device staging,
        outputs, pinned host outputs and events are allocated once per
        (depth, output shape) and reused across calls, so the steady state
        allocates nothing. A yielded tensor is valid until the generator is
        advanced (its slot is then reused). Each slot carries its own status
        words, copied back with its output: a batch with a bad index raises
        the reference's LookupValidationError (first bad index of THAT batch
        in (lookup, feature, position) order) when its turn to be yielded
        comes."""
        eng = self.engine
        dev = eng.device
        st = self._stream_state(depth)
        s_in, s_cmp, s_out = st["streams"]
        slots = st["slots"]
        pending = []

        def launch(bh, k):
            sl = slots[k]
            nnz, nb = int(bh.indices.numel()), int(bh.offsets.numel())
            B = bh.batch_size
            odim = eng.out_dim(bh)
            if (sl["idx"] is None or sl["idx"].numel() < nnz or sl["idx"].dtype != bh.indices.dtype
                    or sl["offs"].numel() < nb or tuple(sl["out"].shape) != (B, odim)):
                torch.cuda.synchronize(dev)  # (re)size the slot: nothing of it may still be in flight
                sl["idx"] = torch.empty(max(nnz, 1) + nnz // 8, dtype=bh.indices.dtype, device=dev)
                sl["offs"] = torch.empty(nb, dtype=torch.int64, device=dev)
                sl["out"] = torch.empty((B, odim), dtype=torch.float32, device=dev)
                sl["host"] = torch.empty((B, odim), dtype=torch.float32, pin_memory=True)
                sl["used"] = False
            with torch.cuda.stream(s_in):
                if sl["used"]:
                    s_in.wait_event(sl["ev_cmp"])  # the slot's device inputs are no longer read
                sl["idx"][:nnz].copy_(bh.indices, non_blocking=True)
                sl["offs"][:nb].copy_(bh.offsets, non_blocking=True)
                sl["ev_in"].record(s_in)
            if "status" not in sl:
                sl["status"] = _lib.Status(dev)
                sl["code_h"] = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(sl["ev_in"])
                if sl["used"]:
                    s_cmp.wait_event(sl["ev_out"])  # the slot's device output was copied out
                dbatch = CsrBatch(sl["idx"][:nnz], sl["offs"][:nb], bh.feature_tables, bh.feature_ops, B)
                sl["batch"] = dbatch
                sl["host_batch"] = bh
                sl["status"].reset()
                eng.pool(dbatch, out=sl["out"], check=False, stream=s_cmp, status=sl["status"])
                sl["ev_cmp"].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(sl["ev_cmp"])
                sl["host"].copy_(sl["out"], non_blocking=True)
                sl["code_h"].copy_(sl["status"].code, non_blocking=True)
                sl["ev_out"].record(s_out)
            sl["used"] = True

        def take(kk, idx_batch):
            sl = slots[kk]
            sl["ev_out"].synchronize()
            if int(sl["code_h"][0]):
                best = eng._first_bad(sl["host_batch"])
                if best is not None:
                    s_, _f, index, t, n = best
                    raise LookupValidationError(f"batch {idx_batch}, lookup {s_}: index {index} out of range "
                                                f"[0,{n}) for table {t}")
                raise LookupValidationError(f"batch {idx_batch}: an index was out of range")
            return sl["host"]

        i = 0
        for bh in batches_host:
            k = i % depth
            if len(pending) == depth:
                kk, bi = pending.pop(0)
                yield take(kk, bi)
            launch(bh, k)
            pending.append((k, i))
            i += 1
        while pending:
            kk, bi = pending.pop(0)
            yield take(kk, bi)
        torch.cuda.synchronize(dev)
