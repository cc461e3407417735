"""Pooling semantics (mirror of embserve/pooling.py) on the GPU.

Contract (pooling.py:1-15): partials carry (sum, count), Mean divides once
at the end; accumulation is f64 in a fixed order (partials by ascending
source, then raw vectors in request order), rounded to f32 on emit. Here the
arithmetic runs in libflexemb kernels (K4 fx_gather_pool, K5 fx_combine);
host code only plans and marshals.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import Enum
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import EmbServeError


class PoolingOp(Enum):
    SUM = "sum"
    MEAN = "mean"


class PlanMode(Enum):
    PUSHDOWN = "pushdown"
    RAW_FETCH = "raw_fetch"


def op_code(op) -> int:
    if isinstance(op, PoolingOp):
        op = op.value
    if op == "sum":
        return _lib.FX_OP_SUM
    if op == "mean":
        return _lib.FX_OP_MEAN
    raise EmbServeError(f"unknown pooling op {op!r}")


@dataclass(frozen=True)
class PartialResult:
    """Shard-side partial pool: f64-accumulated sum emitted as f32, plus the
    number of rows that went in (pooling.py:35-47)."""

    vector: object
    count: int
    source: int = 0

    def __post_init__(self):
        if self.count < 1:
            raise EmbServeError("PartialResult.count must be >= 1")


@dataclass
class PoolingPlan:
    """Pushdown-vs-raw decision per (server, feature position) (pooling.py:49-57)."""

    threshold: int
    modes: dict = field(default_factory=dict)

    def mode(self, server_id: int, feature_pos: int) -> PlanMode:
        return self.modes[(server_id, feature_pos)]


def plan_hierarchical(group_sizes: dict, threshold: int) -> PoolingPlan:
    """Group of size >= threshold is pushed down, smaller groups are raw-fetched
    (pooling.py:88-100). Host-side scalar planning."""
    if threshold < 2:
        raise EmbServeError(f"pushdown threshold must be >= 2, got {threshold}")
    plan = PoolingPlan(threshold=threshold)
    for key, size in group_sizes.items():
        plan.modes[key] = PlanMode.PUSHDOWN if size >= threshold else PlanMode.RAW_FETCH
    return plan


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _as_rows(vectors, dim_check: bool, what: str) -> torch.Tensor:
    """Stack a list of 1-D vectors (numpy or torch) into a [n, D] f32 CUDA tensor."""
    if isinstance(vectors, torch.Tensor):
        t = vectors
        if t.dim() == 1:
            t = t.unsqueeze(0)
        return t.to(device=_device(), dtype=torch.float32).contiguous()
    if isinstance(vectors, np.ndarray) and vectors.ndim == 2:
        return torch.from_numpy(np.ascontiguousarray(vectors, dtype=np.float32)).to(_device())
    dims = {int(np.shape(v)[-1]) for v in vectors}
    if dim_check and len(dims) > 1:
        raise EmbServeError(f"{what}: dim mismatch ({sorted(dims)[1]} != {sorted(dims)[0]})")
    host = np.stack([np.asarray(v.detach().cpu() if isinstance(v, torch.Tensor) else v, dtype=np.float32)
                     for v in vectors])
    return torch.from_numpy(host).to(_device())


def _like_input(example, out: torch.Tensor):
    if isinstance(example, torch.Tensor):
        return out
    return out.cpu().numpy()


def combine_rows_device(partials: torch.Tensor | None, counts: torch.Tensor | None, raw: torch.Tensor | None,
                        op) -> torch.Tensor:
    """One bag: fold f64 partial rows [n_src, D] (already in ascending source
    order) then f32 raw rows [n_raw, D] in order, f64, round once (K5)."""
    dev = _device()
    D = (partials if partials is not None else raw).shape[-1]
    n_src = 0 if partials is None else partials.shape[0]
    out = torch.empty((1, D), dtype=torch.float32, device=dev)
    ptrs = cnts = None
    if n_src:
        partials = partials.to(device=dev, dtype=torch.float64).contiguous()
        counts = counts.to(device=dev, dtype=torch.int32).contiguous()
        ptrs = torch.tensor([partials.data_ptr() + s * D * 8 for s in range(n_src)], dtype=torch.int64, device=dev)
        cnts = torch.tensor([counts.data_ptr() + s * 4 for s in range(n_src)], dtype=torch.int64, device=dev)
    raw_off = None
    if raw is not None and raw.shape[0]:
        raw = raw.to(device=dev, dtype=torch.float32).contiguous()
        raw_off = torch.tensor([0, raw.shape[0]], dtype=torch.int64, device=dev)
    st = _lib.Status(dev)
    _lib.check(_lib.lib.fx_combine(_lib.ptr(ptrs), 0, _lib.ptr(cnts), n_src, D, _lib.ptr(raw_off),
                                   _lib.ptr(raw) if raw_off is not None else None, 1, D, op_code(op), None,
                                   out.data_ptr(), D, st.code.data_ptr(), _lib.stream_ptr()), "combine")
    code, _ = st.read()
    if code:
        raise EmbServeError("combine_partials: nothing to combine")
    return out[0]


def sum_rows_f64(rows, dim: int | None = None):
    """Sequential element-wise sum in input order with an f64 accumulator
    (pooling.py:60-71), computed by K4 in FX_OUT_F64_PARTIAL mode."""
    if len(rows) == 0:
        if dim is None:
            raise EmbServeError("cannot sum zero rows without a dim")
        return np.zeros(dim, dtype=np.float64)
    t = _as_rows(rows, True, "sum_rows_f64")
    out = pool_rows_device(t, op=PoolingOp.SUM, partial=True)
    return _like_input(rows if isinstance(rows, torch.Tensor) else None, out)


def pool_rows_device(rows: torch.Tensor, op, partial: bool = False) -> torch.Tensor:
    """Pool all rows of a [n, D] CUDA tensor as one bag via K4."""
    from .store import pool_csr_device
    n, D = rows.shape
    idx = torch.arange(n, dtype=torch.int32, device=rows.device)
    offs = torch.tensor([0, n], dtype=torch.int64, device=rows.device)
    out = pool_csr_device(rows, 0, n, idx, offs, op, partial=partial)
    return out[0]


def pool_flat(vectors: Sequence, op: PoolingOp):
    """Reduce a non-empty list of equal-dim vectors to one f32 vector
    (pooling.py:74-85): f64 sequential sum, Mean divides once."""
    if len(vectors) == 0:
        raise EmbServeError("pool_flat: empty vector list")
    t = _as_rows(vectors, True, "pool_flat")
    return _like_input(vectors[0] if not isinstance(vectors, torch.Tensor) else vectors,
                       pool_rows_device(t, op))


def combine_partials(partials: Sequence[PartialResult], raw: Sequence, op: PoolingOp):
    """Global pooling step (pooling.py:103-123): partials folded by ascending
    source, then raw vectors in request order, f64, Mean divides by
    (sum of counts + raw count) once; emitted as f32. Runs in K5."""
    if len(partials) == 0 and len(raw) == 0:
        raise EmbServeError("combine_partials: nothing to combine")
    dims = {int(np.shape(p.vector)[-1]) for p in partials} | {int(np.shape(v)[-1]) for v in raw}
    if len(dims) != 1:
        raise EmbServeError(f"combine_partials: inconsistent dims {sorted(dims)}")
    ordered = sorted(partials, key=lambda p: p.source)
    ptens = ctens = None
    if ordered:
        ptens = _as_rows([p.vector for p in ordered], False, "combine_partials").to(torch.float64)
        ctens = torch.tensor([p.count for p in ordered], dtype=torch.int32)
    rtens = _as_rows(list(raw), False, "combine_partials") if len(raw) else None
    out = combine_rows_device(ptens, ctens, rtens, op)
    example = ordered[0].vector if ordered else raw[0]
    return _like_input(example, out)
