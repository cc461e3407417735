"""Range routing (mirror of embserve/routing.py).

The table is built once from the placement and mirrored on the device
(route_off / starts / shard ids / num_rows) so fx_route (K1) resolves whole
batches in one launch. `resolve` (one index, with the comparison-counter
hook the reference tests use, routing.py:66-85) stays a host-side ordered
search; `resolve_many` and `group_by_server` run on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, LookupValidationError
from .store import ShardSpec, TableMeta, validate_placement


@dataclass
class GroupItem:
    """One feature's indices routed to one server and their original
    positions in the feature (routing.py:24-32)."""

    feature_pos: int
    table_id: int
    indices: list
    positions: list


@dataclass
class DestinationGroup:
    server_id: int
    items: list = field(default_factory=list)

    def total_indices(self) -> int:
        return sum(len(it.indices) for it in self.items)


class RoutingTable:
    def __init__(self, metas: dict, shards_by_table: dict):
        # shards_by_table: table -> list[ShardSpec] sorted by start
        self._metas = metas
        self._shards = shards_by_table
        self._dev: dict = {}
        # global shard numbering (table-major, then start): the device routes
        # to shard ids; shard -> server map recovers the reference's server.
        self.shard_list: list = []
        for t in sorted(shards_by_table):
            self.shard_list.extend(shards_by_table[t])
        self.shard_server = np.array([s.server_id for s in self.shard_list], dtype=np.int64)

    def table_ids(self) -> list:
        return sorted(self._shards)

    def entries(self, table_id: int) -> list:
        sh = self._routes(table_id)
        return [(s.start, s.end, s.server_id) for s in sh]

    def _routes(self, table_id: int):
        try:
            return self._shards[table_id]
        except KeyError:
            raise LookupValidationError(f"unknown table {table_id}") from None

    def num_rows(self, table_id: int) -> int:
        self._routes(table_id)
        return self._metas[table_id].num_rows

    def resolve(self, table_id: int, index: int, counter: list | None = None) -> int:
        """Server hosting `index`: rightmost shard start <= index, binary search
        (routing.py:66-85); `counter` accumulates comparisons."""
        sh = self._routes(table_id)
        n = self._metas[table_id].num_rows
        if not (0 <= index < n):
            raise LookupValidationError(f"index {index} out of range [0,{n}) for table {table_id}")
        lo, hi = 0, len(sh)
        while lo < hi:
            mid = (lo + hi) // 2
            if counter is not None:
                counter[0] += 1
            if sh[mid].start <= index:
                lo = mid + 1
            else:
                hi = mid
        return int(sh[lo - 1].server_id)

    # -- device mirror ------------------------------------------------------------

    def device_tables(self, device) -> dict:
        """route_off[t..t+1] spans table t's shard starts; shard_id is the global
        shard number (index into shard_list)."""
        device = torch.device(device)
        key = str(device)
        if key not in self._dev:
            n_t = (max(self._shards) + 1) if self._shards else 0
            route_off = np.zeros(n_t + 1, np.int64)
            starts, sid, nrows = [], [], np.zeros(max(n_t, 1), np.int64)
            gid = 0
            for t in range(n_t):
                sh = self._shards.get(t, [])
                route_off[t + 1] = route_off[t] + len(sh)
                for s in sh:
                    starts.append(s.start)
                    sid.append(self.shard_list.index(s))
                if t in self._metas:
                    nrows[t] = self._metas[t].num_rows
            self._dev[key] = dict(
                route_off=torch.from_numpy(route_off).to(device),
                starts=torch.tensor(starts, dtype=torch.int64, device=device),
                shard_id=torch.tensor(sid, dtype=torch.int32, device=device),
                num_rows=torch.from_numpy(nrows).to(device),
                n_tables=n_t,
            )
        return self._dev[key]

    def route_csr(self, bag_table: torch.Tensor, indices: torch.Tensor, offsets: torch.Tensor,
                  want_dest: bool = True, status: _lib.Status | None = None):
        """K1 over a CSR batch: global shard id per occurrence (int32), or only
        validation when want_dest is False. Returns (dest, status)."""
        dev = indices.device
        dt = self.device_tables(dev)
        st = status or _lib.Status(dev)
        dest = torch.empty(indices.numel(), dtype=torch.int32, device=dev) if want_dest else None
        n_bags = offsets.numel() - 1
        _lib.check(_lib.lib.fx_route(dt["route_off"].data_ptr(), dt["starts"].data_ptr(), dt["shard_id"].data_ptr(),
                                     dt["num_rows"].data_ptr(), bag_table.data_ptr(), indices.data_ptr(),
                                     _lib.idx_type_of(indices), offsets.data_ptr(), n_bags, _lib.ptr(dest),
                                     st.err.data_ptr(), st.code.data_ptr(), _lib.stream_ptr()), "route")
        return dest, st

    def resolve_many(self, table_id: int, indices) -> np.ndarray:
        """Vectorised resolve (routing.py:87-97), one fx_route launch."""
        sh = self._routes(table_id)
        n = self._metas[table_id].num_rows
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        if idx.size == 0:
            return np.zeros(0, dtype=np.int64)
        dev = torch.device("cuda", torch.cuda.current_device())
        ix = torch.from_numpy(idx).to(dev)
        bt = torch.tensor([table_id], dtype=torch.int32, device=dev)
        offs = torch.tensor([0, idx.size], dtype=torch.int64, device=dev)
        dest, st = self.route_csr(bt, ix, offs)
        code, pos = st.read()
        if code:
            bad = int(idx[(idx < 0) | (idx >= n)][0])
            raise LookupValidationError(f"index {bad} out of range [0,{n}) for table {table_id}")
        return self.shard_server[dest.cpu().numpy()]


def build_routing(metas: list, placement: list) -> RoutingTable:
    """Immutable routing table from a valid placement (routing.py:100-114)."""
    meta_map = {m.table_id: m for m in metas}
    if len(meta_map) != len(metas):
        raise ConfigError("duplicate table_id in metas")
    validate_placement(meta_map, placement)
    by_table = {t: sorted((s for s in placement if s.table_id == t), key=lambda s: s.start) for t in meta_map}
    return RoutingTable(meta_map, by_table)


def group_by_server(rt: RoutingTable, lookup) -> list:
    """Partition a lookup's indices by destination server, order-preserving,
    groups sorted by server id (routing.py:117-148). Routing runs on the GPU
    (one fx_route over all features); the Python group objects are assembled
    from its output."""
    feats = lookup.features
    dev = torch.device("cuda", torch.cuda.current_device())
    lens = [len(f.indices) for f in feats]
    for pos, f in enumerate(feats):
        if f.table_id not in rt._shards:
            raise LookupValidationError(f"feature {pos} (table {f.table_id}): unknown table {f.table_id}")
    idx = np.concatenate([np.asarray(f.indices, dtype=np.int64) for f in feats]) if feats else np.zeros(0, np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bt = torch.tensor([f.table_id for f in feats], dtype=torch.int32, device=dev)
    dest, st = rt.route_csr(bt, torch.from_numpy(idx).to(dev), torch.from_numpy(offs).to(dev))
    code, pos = st.read()
    if code:
        fpos = int(np.searchsorted(offs, pos, side="right") - 1)
        f = feats[fpos]
        n = rt.num_rows(f.table_id)
        bad = int(idx[pos])
        raise LookupValidationError(
            f"feature {fpos} (table {f.table_id}): index {bad} out of range [0,{n}) for table {f.table_id}")
    servers = rt.shard_server[dest.cpu().numpy()]
    groups: dict = {}
    for fp, f in enumerate(feats):
        srv = servers[offs[fp]:offs[fp + 1]]
        items: dict = {}
        for i, (index, s) in enumerate(zip(f.indices, srv)):
            item = items.get(int(s))
            if item is None:
                item = items[int(s)] = GroupItem(feature_pos=fp, table_id=f.table_id, indices=[], positions=[])
            item.indices.append(index)
            item.positions.append(i)
        for s, item in items.items():
            groups.setdefault(s, DestinationGroup(server_id=s)).items.append(item)
    return [groups[s] for s in sorted(groups)]
