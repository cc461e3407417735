"""HBM-resident sharded embedding store (mirror of embserve/store.py).

Shards are row-major [end-start, dim] f32 CUDA tensors materialised on the
GPU by K0 (fx_table_init) from the reference PRF, bit-identical to
store.py:62-89. Raw gathers (lookup_rows) and server-side partial pooling
(partial_pool) run in libflexemb kernels; the legacy per-feature methods
return fresh numpy arrays like the reference (store.py:166).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, EmbServeError, RoutingViolationError
from .pooling import PartialResult, PoolingOp, op_code
from .wire import ELEMENT_WIDTH


@dataclass(frozen=True)
class TableMeta:
    table_id: int
    num_rows: int
    dim: int
    element_width: int = ELEMENT_WIDTH

    def __post_init__(self):
        if self.num_rows < 1:
            raise ConfigError(f"table {self.table_id}: num_rows must be >= 1")
        if self.dim < 1:
            raise ConfigError(f"table {self.table_id}: dim must be >= 1")
        if self.element_width != ELEMENT_WIDTH:
            raise ConfigError(f"table {self.table_id}: element_width is fixed at {ELEMENT_WIDTH}")

    @property
    def row_bytes(self) -> int:
        return self.dim * self.element_width


@dataclass(frozen=True)
class ShardSpec:
    """Rows [start, end) of one table on one server (store.py:43-50)."""

    table_id: int
    start: int
    end: int
    server_id: int


@dataclass
class Shard:
    table_id: int
    start: int
    end: int
    host: int
    data: torch.Tensor | None  # [end-start, dim] f32 on the owning GPU; None if remote


def _device(device=None) -> torch.device:
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def table_block_device(seed: int, table_id: int, dim: int, start: int, end: int, device=None,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """K0: rows [start, end) of table `table_id` as a CUDA tensor (store.py:82-89)."""
    dev = _device(device)
    n = end - start
    if out is None:
        out = torch.empty((n, dim), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib.fx_table_init(out.data_ptr(), out.stride(0), seed % (1 << 64), table_id, dim, start, n,
                                          _lib.stream_ptr()), "table_init")
    return out


def table_block(seed: int, table_id: int, dim: int, start: int, end: int) -> np.ndarray:
    """Deterministic (end-start, dim) f32 block (store.py:82-89), computed on the GPU."""
    return table_block_device(seed, table_id, dim, start, end).cpu().numpy()


def row_values(seed: int, table_id: int, row: int, dim: int) -> np.ndarray:
    """One row's contents (store.py:77-79)."""
    return table_block(seed, table_id, dim, row, row + 1)[0]


def validate_placement(metas: dict, placement: list) -> None:
    """Shards of every table are disjoint and cover [0, num_rows) (store.py:92-119)."""
    by_table: dict = {}
    for spec in placement:
        if spec.table_id not in metas:
            raise ConfigError(f"placement references unknown table {spec.table_id}")
        if not (0 <= spec.start < spec.end):
            raise ConfigError(f"table {spec.table_id}: invalid shard range [{spec.start},{spec.end})")
        by_table.setdefault(spec.table_id, []).append(spec)
    for table_id, meta in metas.items():
        shards = sorted(by_table.get(table_id, []), key=lambda s: s.start)
        if not shards:
            raise ConfigError(f"table {table_id}: no shards placed, gap [0,{meta.num_rows})")
        if shards[-1].end > meta.num_rows:
            raise ConfigError(f"table {table_id}: shard end {shards[-1].end} beyond {meta.num_rows} rows")
        cursor = 0
        for spec in shards:
            if spec.start < cursor:
                raise ConfigError(f"table {table_id}: overlap at row {spec.start}")
            if spec.start > cursor:
                raise ConfigError(f"table {table_id}: gap [{cursor},{spec.start})")
            cursor = spec.end
        if cursor < meta.num_rows:
            raise ConfigError(f"table {table_id}: gap [{cursor},{meta.num_rows})")


def make_segments(segs: list, device) -> torch.Tensor:
    """Pack fx_segment descriptors into a device byte tensor."""
    arr = (_lib.FxSegment * len(segs))(*segs)
    host = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
    return host.to(device)


def pool_csr_device(table: torch.Tensor, row_begin: int, row_end: int, indices: torch.Tensor,
                    offsets: torch.Tensor, op, partial: bool = False, out: torch.Tensor | None = None,
                    counts: torch.Tensor | None = None, status: _lib.Status | None = None,
                    bad_code: int = _lib.FX_E_ROUTING_VIOLATION) -> torch.Tensor:
    """K4 over one shard: pooled [n_bags, D] (f32 final, or f64 partial sums)."""
    dev = table.device
    n_bags = offsets.numel() - 1
    D = table.shape[1]
    if out is None:
        # partial mode leaves empty bags' rows unwritten (count 0 = partial absent)
        out = (torch.zeros if partial else torch.empty)((n_bags, D), dtype=torch.float64 if partial else torch.float32,
                                                        device=dev)
    _lib.check_out(out, n_bags, D, dtype=torch.float64 if partial else torch.float32)
    esz = 2 if partial else 1   # f64 outputs: 16 B = 2 elements
    aligned = _lib.vec_ok((out.data_ptr(), out.stride(0) * esz), (table.data_ptr(), table.stride(0)))
    seg = _lib.FxSegment(table.data_ptr(), row_begin, row_end, 0, n_bags, out.data_ptr(), out.stride(0),
                         table.stride(0), D, op_code(op))
    segs = make_segments([seg], dev)
    own = status is None
    st = status or _lib.Status(dev)
    _lib.check(_lib.lib.fx_gather_pool(segs.data_ptr(), 1, D, indices.data_ptr(), _lib.idx_type_of(indices),
                                       offsets.data_ptr(), n_bags,
                                       (_lib.FX_OUT_F64_PARTIAL if partial else _lib.FX_OUT_F32)
                                       | (0 if aligned else _lib.FX_OUT_SCALAR),
                                       _lib.ptr(counts), st.err.data_ptr(), bad_code, st.code.data_ptr(),
                                       _lib.stream_ptr()), "gather_pool")
    if own:
        code, pos = st.read()
        if code:
            bad = int(indices[pos].item())
            raise RoutingViolationError(f"row {bad} not hosted by shard [{row_begin},{row_end})")
    return out


class ServerStore:
    """Shards hosted by one server (= one GPU rank in the B200 build)
    (store.py:122-193)."""

    def __init__(self, server_id: int, cpu_budget: int = 16):
        self.server_id = server_id
        self.cpu_budget = cpu_budget
        self._shards: dict = {}
        self._starts: dict = {}

    def add_shard(self, shard: Shard) -> None:
        if shard.host != self.server_id:
            raise ConfigError(f"shard of table {shard.table_id} hosted on {shard.host}, not server {self.server_id}")
        self._shards.setdefault(shard.table_id, []).append(shard)
        self._shards[shard.table_id].sort(key=lambda s: s.start)
        self._starts[shard.table_id] = np.array([s.start for s in self._shards[shard.table_id]], dtype=np.int64)

    def hosted_tables(self) -> list:
        return sorted(self._shards)

    def shards(self, table_id: int) -> list:
        return self._shards.get(table_id, [])

    # -- device paths ---------------------------------------------------------

    def _split(self, table_id: int, idx: np.ndarray):
        """Which hosted shard each index falls in (host control logic, the
        same ordered search as store.py:165); raises like store.py:168-180."""
        shards = self._shards.get(table_id)
        if shards is None:
            raise RoutingViolationError(f"server {self.server_id} hosts no shard of table {table_id}")
        which = np.searchsorted(self._starts[table_id], idx, side="right") - 1
        for s in np.unique(which):
            mask = which == s
            if s < 0:
                bad = int(idx[mask][0])
                raise RoutingViolationError(f"server {self.server_id}: row {bad} of table {table_id} not hosted here")
            rows = idx[mask]
            if rows.max() >= shards[s].end:
                bad = int(rows[rows >= shards[s].end][0])
                raise RoutingViolationError(f"server {self.server_id}: row {bad} of table {table_id} not hosted here")
        return shards, which

    def lookup_rows_device(self, table_id: int, indices) -> torch.Tensor:
        """Gather rows in input order, duplicates per occurrence (store.py:151-182)."""
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        shards, which = self._split(table_id, idx) if idx.size else (self._shards.get(table_id), None)
        if shards is None:
            raise RoutingViolationError(f"server {self.server_id} hosts no shard of table {table_id}")
        D = shards[0].data.shape[1]
        dev = shards[0].data.device
        out = torch.empty((idx.size, D), dtype=torch.float32, device=dev)
        if idx.size == 0:
            return out
        st = _lib.Status(dev)
        for s in np.unique(which):
            sh = shards[s]
            sel = np.nonzero(which == s)[0]
            dst = out if sel.size == idx.size else torch.empty((sel.size, D), dtype=torch.float32, device=dev)
            ix = torch.from_numpy(idx[sel]).to(dev)
            _lib.check(_lib.lib.fx_gather_rows(sh.data.data_ptr(), sh.data.stride(0), sh.start, sh.end, D,
                                               ix.data_ptr(), _lib.FX_IDX_I64, sel.size, dst.data_ptr(),
                                               st.err.data_ptr(), st.code.data_ptr(), _lib.stream_ptr()),
                       "lookup_rows")
            if dst is not out:
                out[torch.from_numpy(sel).to(dev)] = dst
        return out

    def lookup_rows(self, table_id: int, indices) -> np.ndarray:
        return self.lookup_rows_device(table_id, indices).cpu().numpy()

    def partial_pool_device(self, table_id: int, indices, op: PoolingOp):
        """(f32 sum of the selected rows accumulated in f64 in input order,
        count) (store.py:184-193)."""
        if len(indices) == 0:
            raise EmbServeError("empty partial pool")
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        shards, which = self._split(table_id, idx)
        dev = shards[0].data.device
        if np.all(which == which[0]):
            sh = shards[which[0]]
            ix = torch.from_numpy(idx).to(dev)
            offs = torch.tensor([0, idx.size], dtype=torch.int64, device=dev)
            vec = pool_csr_device(sh.data, sh.start, sh.end, ix, offs, PoolingOp.SUM)[0]
        else:
            rows = self.lookup_rows_device(table_id, idx)
            from .pooling import pool_rows_device
            vec = pool_rows_device(rows, PoolingOp.SUM)
        return vec, int(idx.size)

    def partial_pool(self, table_id: int, indices, op: PoolingOp) -> PartialResult:
        vec, n = self.partial_pool_device(table_id, indices, op)
        return PartialResult(vector=vec.cpu().numpy(), count=n, source=self.server_id)


@dataclass
class Deployment:
    """All servers of one run, immutable after init_store (store.py:196-225)."""

    metas: dict
    servers: dict
    placement: list
    seed: int
    server_ids: list = field(init=False)

    def __post_init__(self):
        self.server_ids = sorted(self.servers)

    def meta(self, table_id: int) -> TableMeta:
        try:
            return self.metas[table_id]
        except KeyError:
            raise ConfigError(f"unknown table {table_id}") from None

    def shard_for(self, table_id: int, row: int) -> Shard:
        for spec in self.placement:
            if spec.table_id == table_id and spec.start <= row < spec.end:
                server = self.servers.get(spec.server_id)
                if server is None:
                    break
                for sh in server.shards(table_id):
                    if sh.start == spec.start:
                        return sh
        raise ConfigError(f"table {table_id}: row {row} not covered by placement")

    def get_row_device(self, table_id: int, row: int) -> torch.Tensor:
        meta = self.meta(table_id)
        if not (0 <= row < meta.num_rows):
            raise EmbServeError(f"row {row} out of range for table {table_id}")
        sh = self.shard_for(table_id, row)
        if sh.data is None:
            # remote shard: recompute from the PRF on this GPU (store.py:77-79)
            return table_block_device(self.seed, table_id, meta.dim, row, row + 1)[0]
        return sh.data[row - sh.start]

    def get_row(self, table_id: int, row: int) -> np.ndarray:
        """Direct row read regardless of placement (store.py:215-225)."""
        return self.get_row_device(table_id, row).cpu().numpy().copy()


def init_store(metas: list, placement: list, seed: int, cpu_budget: int = 16, device=None,
               hosts=None) -> Deployment:
    """Materialise every shard on the GPU with deterministic contents
    (store.py:228-251). `hosts` (optional set of server ids) limits which
    shards this process materialises — the others are placed on other ranks
    and recorded with data=None."""
    meta_map = {m.table_id: m for m in metas}
    if len(meta_map) != len(metas):
        raise ConfigError("duplicate table_id in metas")
    validate_placement(meta_map, placement)
    dev = _device(device)
    servers: dict = {}
    for spec in placement:
        meta = meta_map[spec.table_id]
        server = servers.setdefault(spec.server_id, ServerStore(spec.server_id, cpu_budget))
        data = None
        if hosts is None or spec.server_id in hosts:
            data = table_block_device(seed, spec.table_id, meta.dim, spec.start, spec.end, device=dev)
        server.add_shard(Shard(table_id=spec.table_id, start=spec.start, end=spec.end, host=spec.server_id, data=data))
    return Deployment(metas=meta_map, servers=servers, placement=list(placement), seed=seed)
