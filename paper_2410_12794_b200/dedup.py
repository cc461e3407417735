"""Per-batch index dedup (K2, fx_dedup): the spatial-locality layer.

No reference counterpart; parity target is
np.unique(table << 40 | row, return_inverse, return_counts). The kernel
hashes every occurrence's 64-bit key, then assigns unique ids in
first-occurrence (lookup, feature, position) order — the order the
reference's per-batch offer dict uses (ranker.py:340) — so its output is
deterministic; sorting `uniq` gives np.unique's order exactly.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib


@dataclass
class DedupResult:
    uniq: torch.Tensor       # u64 keys as int64 [n_uniq], first-occurrence order
    mult: torch.Tensor       # int32 [n_uniq]
    first_ord: torch.Tensor  # int64 [n_uniq] sample-major ordinal of the first occurrence
    last_ord: torch.Tensor   # int64 [n_uniq] ... of the last occurrence
    inverse: torch.Tensor    # int32 [nnz] unique id per occurrence (CSR order)
    n_uniq: int


def sample_major_starts(offsets: torch.Tensor, batch_size: int, n_features: int) -> torch.Tensor:
    """sm_start[b] for table-major bags b = f*B + s: the (lookup, feature)
    ordinal of the bag's first index, i.e. the exclusive prefix of bag lengths
    in (sample, feature) order (ranker.py:227-235 probe order)."""
    lens = (offsets[1:] - offsets[:-1]).view(n_features, batch_size).t().reshape(-1)
    ex = torch.cumsum(lens, 0) - lens
    return ex.view(batch_size, n_features).t().reshape(-1).contiguous()


class Deduper:
    """Owns the reusable workspace for fx_dedup."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.ws = None

    def __call__(self, bag_table, indices, offsets, sm_start, nnz=None, sync=True) -> DedupResult:
        dev = indices.device
        n_bags = offsets.numel() - 1
        nnz = int(indices.numel()) if nnz is None else nnz
        need = ctypes.c_size_t(0)
        _lib.check(_lib.lib.fx_dedup(None, None, 0, None, None, n_bags, nnz, None, None, None, None, None, None,
                                     None, ctypes.byref(need), None), "dedup")
        if self.ws is None or self.ws.numel() < need.value:
            self.ws = torch.empty(need.value, dtype=torch.uint8, device=dev)
        uniq = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        mult = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        fo = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        lo = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        inv = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        nu = torch.zeros(1, dtype=torch.int64, device=dev)
        wsb = ctypes.c_size_t(self.ws.numel())
        _lib.check(_lib.lib.fx_dedup(bag_table.data_ptr(), indices.data_ptr(), _lib.idx_type_of(indices),
                                     offsets.data_ptr(), sm_start.data_ptr(), n_bags, nnz, uniq.data_ptr(),
                                     mult.data_ptr(), fo.data_ptr(), lo.data_ptr(), inv.data_ptr(), nu.data_ptr(),
                                     self.ws.data_ptr(), ctypes.byref(wsb), _lib.stream_ptr()), "dedup")
        n = int(nu.item()) if sync else -1
        if sync:
            uniq, mult, fo, lo = uniq[:n], mult[:n], fo[:n], lo[:n]
        return DedupResult(uniq, mult, fo, lo, inv[:nnz], n)


def dedup_csr(bag_table, indices, offsets, batch_size, n_features) -> DedupResult:
    sm = sample_major_starts(offsets, batch_size, n_features)
    return Deduper(indices.device)(bag_table, indices, offsets, sm)
