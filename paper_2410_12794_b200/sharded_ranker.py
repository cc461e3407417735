"""The Ranker pipeline (ranker.py) on every GPU of a sharded deployment.

Each rank is a ranker with its OWN cache ("each requester GPU
keeps its own cache"; multi-GPU cache partitioning is a reference non-goal,
SPEC.md:312) over a store sharded across the ranks. Per batch it runs the
single-GPU pipeline of `Ranker` unchanged — validation, apply_pending,
admission check, pooled-result probe, dedup + row probe, plan, counters,
offers, maintenance (ranker.py:218-442) — and only the pooling step is
distributed (`P2PShardedLookup.pool_cached`): cache hits are combined from
the requester's cache rows, groups of at least `pushdown_threshold` misses
per (bag, owner) are pushed down to the owner's K4 (partial into the
requester's buffer over NVLink), smaller groups are raw-fetched with peer
loads from the owner's shard, and K5 folds partials (ascending owner) then
raw vectors (cache hits and raw fetches, position order) — combine_partials'
order (pooling.py:103-123). Offers and staged admissions read their rows
from the owners' shards over NVLink (the cache's table directory holds the
IPC-mapped shard pointers), the analogue of `Deployment.get_row`.

All ranks call `execute_csr` in lockstep (one batch each per step).
"""

from __future__ import annotations

import torch

from . import _lib
from .dedup import Deduper
from .errors import ConfigError
from .ranker import Ranker, RankerParams
from .routing import build_routing
from .sharded import P2PShardedLookup
from .store import Deployment, ServerStore, Shard

_NO_PUSHDOWN = (1 << 31) - 1  # threshold None: every group raw-fetched (ranker.py:270-271)


class ShardedRanker(Ranker):
    def __init__(self, metas, placement, seed: int, rank: int, world: int, device, feature_tables, feature_ops,
                 batch_size: int, params: RankerParams | None = None, cache=None, policy=None, tracker=None,
                 group=None, partial_dtype: str = "f64", max_nnz: int | None = None):
        params = params or RankerParams()
        thr = params.pushdown_threshold
        if thr is not None and thr < 2:
            raise ConfigError(f"pushdown threshold must be >= 2, got {thr}")
        self.device = torch.device(device)
        self.sl = P2PShardedLookup(metas, placement, seed, feature_tables, feature_ops, batch_size, rank, world,
                                   self.device, group=group, mode="rowwise", max_nnz=max_nnz,
                                   partial_dtype=partial_dtype,
                                   pushdown_threshold=_NO_PUSHDOWN if thr is None else thr)
        meta_map = {m.table_id: m for m in metas}
        servers = {}
        for sp in placement:
            srv = servers.setdefault(sp.server_id, ServerStore(sp.server_id))
            data = self.sl.ops.local[sp.table_id][0] if sp.server_id == rank else None
            srv.add_shard(Shard(sp.table_id, sp.start, sp.end, sp.server_id, data))
        self.deployment = Deployment(metas=meta_map, servers=servers, placement=list(placement), seed=seed)
        self.routing = build_routing(metas, placement)
        self.transport = None
        self.params = params
        self.cache, self.policy, self.tracker = cache, policy, tracker
        self.batch_metrics, self.results = [], {}
        self._last_level = None
        self._dedup = Deduper(self.device)
        self._status = _lib.Status(self.device)
        self._shards = []
        self._server_ids = sorted({sp.server_id for sp in placement})
        self._shard_server_dev = torch.tensor([self._server_ids.index(sp.server_id)
                                               for sp in self.routing.shard_list], dtype=torch.int64,
                                              device=self.device)
        self._single_shard, self._table_shard = False, {}
        self.hits_from_cache = True
        self.profile, self.stage_ms, self._marks = False, {}, []
        self._init_fast_state(False)  # the sharded pooling runs the staged pipeline
        self._occ_slot = None
        self.ftab, self.B = tuple(feature_tables), batch_size
        if cache is not None:
            # every shard, local or a peer's (IPC-mapped), is an admission source
            bases = self.sl.t_shard_base.cpu().tolist()
            dirs = []
            for sp, base in zip(self.sl.ops.shard_list, bases):
                D = meta_map[sp.table_id].dim
                dirs.append((base, sp.start, sp.end, D, sp.table_id, D))
            cache.bind_dir(dirs)

    def execute_batch(self, batch):
        raise ConfigError("ShardedRanker takes fixed-shape CSR batches: use execute_csr")

    def execute_csr(self, indices, offsets, feature_tables=None, feature_ops=None, batch_size=None, batch_id=0):
        ft = tuple(feature_tables) if feature_tables is not None else self.ftab
        if ft != self.ftab or (batch_size is not None and batch_size != self.B):
            raise ConfigError("ShardedRanker batches must match the configured features and batch size")
        return super().execute_csr(indices, offsets, self.ftab, feature_ops or self.sl.fops, self.B, batch_id)

    def _pool(self, lay, dest, hit_occ, dd, nnz, n_bags) -> torch.Tensor:
        hit_slot = self._occ_slot.to(torch.int32).contiguous() if self._occ_slot is not None else None
        out = self.sl.pool_cached(lay.indices, lay.offsets, hit_slot, self.cache)
        return out.clone()

    def counters(self) -> torch.Tensor:
        return self.sl.counters()
