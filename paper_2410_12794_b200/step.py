"""Fused, sync-free per-batch cache step (csrc/fx_step.cu) behind the Ranker.

`BatchStep` binds one AdaptiveCache and the deployment's HBM-resident tables
to the fx_step_* entry points (include/flexemb.h). One `run` enqueues the
whole locality layer of a batch — apply_pending_admissions, ingress
validation, dedup, probe, pushdown plan + per-bag counters, ordered offers —
and `maintain` enqueues stage_hot_admissions(limit) + sketch age, in the
reference's order (ranker.py:218-442, cache.py:189-352). Neither call
synchronises with the host, so a Ranker batch can be captured as a CUDA
graph; device-side errors are read back with `scalars()` (one sync).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import CapacityError, ConfigError, InvariantError

# StepScalars field order (csrc/fx_step.cu)
SCALARS = ("err", "err_at", "epoch", "n_uniq", "n_cand", "n_hitu", "n_nonhit", "n_hard", "n_rej", "n_off", "e0",
           "F", "mode", "n_acc", "n_ev", "ftop0", "log0", "tick0", "tick_base", "minc_bits", "b_hits", "b_misses",
           "b_groups", "b_applied", "b_pd_groups", "b_pd_rows", "b_raw_rows", "rebuild_index", "rehash_sketch",
           "rehash_n", "stage_on", "topk_live", "topk_krem", "topk_n", "topk_hi", "topk_lo", "topk_digit", "qlen_new", "n_levels", "codes_on", "chain_cycles", "dyn", "claim_tag", "claim_clear",
           "dedup_merge", "stage_thr", "topk_fast")
IDX = {k: i for i, k in enumerate(SCALARS)}
ERR_BAD_INDEX, ERR_SKETCH_CAP, ERR_INVARIANT = 1, 2, 3


def _sig():
    L = _lib.lib
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sigs = {
        "fx_step_create": ([ctypes.POINTER(P), P, I64, I64, P, P, P, I32, I32, I64, I32], ctypes.c_int),
        "fx_step_destroy": ([P], ctypes.c_int),
        "fx_step_prepare": ([P, P], ctypes.c_int),
        "fx_step_start": ([P, I32, P, P, I32, P, P, I64, I64, I32, P, P, P, P, P], ctypes.c_int),
        "fx_step_offer": ([P, I32, P], ctypes.c_int),
        "fx_step_maintain": ([P, I32, I64, I32, P], ctypes.c_int),
        "fx_step_join": ([P, P], ctypes.c_int),
        "fx_step_scalars": ([P, I32, P, I64, P], ctypes.c_int),
        "fx_step_scalars_device": ([P, I32], P),
        "fx_step_launches": ([P], I64),
    }
    for n, (a, r) in sigs.items():
        f = getattr(L, n)
        f.argtypes = a
        f.restype = r
    return L


class BatchStep:
    """Device state of the fused step for one cache over one deployment.

    Domain: every table one shard on this GPU with one row size (= the
    cache's entry size), row keys only (no pooled-result keyspace)."""

    def __init__(self, cache, deployment, max_nnz: int, max_bags: int, stage_limit_cap: int = 64, slots: int = 1):
        if cache.pooled_results_enabled:
            raise ConfigError("the fused step handles row keys only (pooled_results off)")
        self._L = _sig()
        self.cache = cache
        self.device = cache.device
        dims = {m.dim for m in deployment.metas.values()}
        if len(dims) != 1:
            raise ConfigError("the fused step needs one row size for every table")
        self.dim = dims.pop()
        n_t = max(deployment.metas) + 1
        base = (ctypes.c_void_p * n_t)()
        ld = (ctypes.c_int64 * n_t)()
        rows = (ctypes.c_int64 * n_t)(*([-1] * n_t))   # absent table ids: every index is out of range
        self._keep = []
        for t, m in deployment.metas.items():
            sh = None
            for server in deployment.servers.values():
                for s in server.shards(t):
                    if s.data is not None and s.data.device == self.device and s.start == 0 and s.end == m.num_rows:
                        sh = s
            if sh is None:
                raise ConfigError(f"table {t} is not one shard resident on {self.device}")
            base[t] = sh.data.data_ptr()
            ld[t] = sh.data.stride(0)
            rows[t] = m.num_rows
            self._keep.append(sh.data)
        self.max_nnz, self.max_bags = int(max_nnz), int(max_bags)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._L.fx_step_create(ctypes.byref(h), cache._h, self.max_nnz, self.max_bags, base, ld, rows,
                                              n_t, self.dim, int(stage_limit_cap), int(slots)), "step create")
        self._h = h
        self.n_slots = int(slots)
        self.tk_cap = max(cache.capacity()["sketch"], cache.capacity()["slots"])
        self.stage_limit_cap = int(stage_limit_cap)
        self.slots = cache._slots

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self._L.fx_step_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def prepare(self, stream=None) -> None:
        """(Re)build the LRU queue if another entry point moved entries."""
        _lib.check(self._L.fx_step_prepare(self._h, _lib.stream_ptr(stream)), "step prepare")

    def start(self, slot: int, bag_table, indices, offsets, sm_start, n_bags: int, nnz: int, threshold, hits_bag,
              pd_groups, pd_rows, raw_rows, stream=None) -> None:
        """apply_pending -> validation + dedup -> probes -> plan + per-bag counters."""
        thr = 0 if threshold is None else int(threshold)
        _lib.check(self._L.fx_step_start(self._h, int(slot), bag_table.data_ptr(), indices.data_ptr(),
                                         _lib.idx_type_of(indices), offsets.data_ptr(), sm_start.data_ptr(),
                                         int(n_bags), int(nnz), thr, _lib.ptr(hits_bag), _lib.ptr(pd_groups),
                                         _lib.ptr(pd_rows), _lib.ptr(raw_rows), _lib.stream_ptr(stream)), "step start")

    def offer(self, slot: int, stream=None) -> None:
        """Ordered offers of the slot's raw-fetched misses."""
        _lib.check(self._L.fx_step_offer(self._h, int(slot), _lib.stream_ptr(stream)), "step offer")

    def maintain(self, slot: int, stage_limit: int, age: bool, stream=None) -> None:
        """stage_hot_admissions(stage_limit) then sketch age."""
        _lib.check(self._L.fx_step_maintain(self._h, int(slot), int(stage_limit), 1 if age else 0,
                                            _lib.stream_ptr(stream)), "step maintain")

    def join(self, stream=None) -> None:
        """Order `stream` after the step's side-stream row copies."""
        _lib.check(self._L.fx_step_join(self._h, _lib.stream_ptr(stream)), "step join")

    def scalars(self, slot: int = 0, stream=None) -> dict:
        """[sync] a slot's device scalars."""
        out = (ctypes.c_int64 * len(SCALARS))()
        _lib.check(self._L.fx_step_scalars(self._h, int(slot), out, len(SCALARS), _lib.stream_ptr(stream)),
                   "step scalars")
        return dict(zip(SCALARS, list(out)))

    def launches(self) -> int:
        """Kernels this step handle launched so far (CUB sweeps count 2)."""
        return int(self._L.fx_step_launches(self._h))

    def scalars_tensor(self, slot: int) -> torch.Tensor:
        """A zero-copy int64 view of a slot's device scalars (async snapshots)."""
        return _dev_view(self._L.fx_step_scalars_device(self._h, int(slot)), len(SCALARS), self.device)

    @staticmethod
    def raise_error(code: int, where: str = "") -> None:
        if code == ERR_SKETCH_CAP:
            raise CapacityError(f"{where}sketch capacity too small for the batch; raise AdaptiveCache(sketch_capacity)")
        if code == ERR_INVARIANT:
            raise InvariantError(f"{where}cache LRU queue out of sync with its entries")
        if code:
            raise InvariantError(f"{where}fused step error {code}")


def _dev_view(ptr: int, n: int, device) -> torch.Tensor:
    """int64[n] tensor aliasing device memory owned by the library."""
    class _Holder:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (int(ptr), False), "version": 3,
                                    "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Holder(), device=device)
