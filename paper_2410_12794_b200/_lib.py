"""ctypes binding of libflexemb.so (include/flexemb.h).

The library is the only compute path: if it is missing this module raises at
import time (no CPU fallback). Device buffers are torch CUDA tensors passed
by data_ptr(); every call runs on torch's current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FX_LIB_PATH", os.path.join(_HERE, "libflexemb.so"))  # override: A/B builds

FX_OK = 0
FX_E_CONFIG = 1
FX_E_LOOKUP_VALIDATION = 2
FX_E_ROUTING_VIOLATION = 3
FX_E_CAPACITY = 4
FX_E_INVARIANT = 5
FX_E_EMPTY = 6
FX_E_CUDA = 7

FX_OP_SUM = 0
FX_OP_MEAN = 1
FX_IDX_I32 = 0
FX_IDX_I64 = 1
FX_OUT_F32 = 0
FX_OUT_F64_PARTIAL = 1
FX_OUT_F32_PARTIAL = 2
FX_OUT_SYSFENCE = 16
FX_OUT_SCALAR = 32
FX_OUT_SHARE = 64

INT64_MAX = (1 << 63) - 1

_CODE_TO_EXC = {
    FX_E_CONFIG: errors.ConfigError,
    FX_E_LOOKUP_VALIDATION: errors.LookupValidationError,
    FX_E_ROUTING_VIOLATION: errors.RoutingViolationError,
    FX_E_CAPACITY: errors.CapacityError,
    FX_E_INVARIANT: errors.InvariantError,
    FX_E_EMPTY: errors.EmbServeError,
    FX_E_CUDA: errors.EmbServeError,
}


class FxSegment(ctypes.Structure):
    """Mirror of `fx_segment` (include/flexemb.h)."""
    _fields_ = [
        ("table", ctypes.c_void_p),
        ("row_begin", ctypes.c_int64),
        ("row_end", ctypes.c_int64),
        ("bag_begin", ctypes.c_int64),
        ("bag_end", ctypes.c_int64),
        ("out", ctypes.c_void_p),
        ("out_stride", ctypes.c_int64),
        ("ld", ctypes.c_int64),
        ("dim", ctypes.c_int32),
        ("op", ctypes.c_int32),
        ("idx", ctypes.c_void_p),
        ("offs", ctypes.c_void_p),
    ]


SEGMENT_BYTES = ctypes.sizeof(FxSegment)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2410_12794_b200/build.py` "
        "(there is no CPU fallback for the lookup path)")

lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_SZP = ctypes.POINTER(ctypes.c_size_t)

_SIGS = {
    "fx_last_error": ([], ctypes.c_char_p),
    "fx_version": ([], ctypes.c_int),
    "fx_num_sms": ([ctypes.c_int], ctypes.c_int),
    "fx_bounds_report": ([ctypes.POINTER(_I64)], ctypes.c_int),
    "fx_bounds_selftest": ([], ctypes.c_int),
    "fx_table_base": ([_U64, _I64], _U64),
    "fx_table_init": ([_P, _I64, _U64, _I64, _I32, _I64, _I64, _P], ctypes.c_int),
    "fx_gather_pool": ([_P, _I32, _I32, _P, _I32, _P, _I64, _I32, _P, _P, _I32, _P, _P], ctypes.c_int),
    "fx_gather_rows": ([_P, _I64, _I64, _I64, _I32, _P, _I32, _I64, _P, _P, _P, _P], ctypes.c_int),
    "fx_combine": ([_P, _I32, _P, _I32, _I64, _P, _P, _I64, _I32, _I32, _P, _P, _I64, _P, _P], ctypes.c_int),
    "fx_route": ([_P, _P, _P, _P, _P, _P, _I32, _P, _I64, _P, _P, _P, _P], ctypes.c_int),
    "fx_bucket": ([_P, _I64, _P, _I64, _I32, _P, _P, _P, _P, _SZP, _P], ctypes.c_int),
    "fx_dedup": ([_P, _P, _I32, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _SZP, _P], ctypes.c_int),
    "fx_dev_alloc": ([ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "fx_dev_free": ([_P], ctypes.c_int),
    "fx_ipc_export": ([_P, ctypes.c_char_p], ctypes.c_int),
    "fx_ipc_open": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "fx_ipc_close": ([_P], ctypes.c_int),
    "fx_can_access_peer": ([ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "fx_memcpy_async": ([_P, _P, ctypes.c_size_t, _P], ctypes.c_int),
    "fx_peer_barrier": ([_P, _P, _I32, _I32, _I64, _P, _P], ctypes.c_int),
    "fx_push_csr": ([_P, _I32, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _I32, _P], ctypes.c_int),
    "fx_rw_push": ([_P, _P, _P, _P, _P, _I32, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZP, _P], ctypes.c_int),
    "fx_rw_push_planned": ([_P, _P, _P, _P, _P, _P, _I32, _P, _I64, _I32, _I32, _P, _P, _P, _P, _P, _I64, _P, _P, _P,
                            _P, _P, _I64, _P, _SZP, _P], ctypes.c_int),
    "fx_combine_ptr": ([_P, _I32, _P, _I32, _I64, _P, _P, _I64, _I32, _I32, _P, _P, _I64, _P, _I64, _P], ctypes.c_int),
    # cache entry points are typed in cache.py (_sig); listed here for export checks
    **{n: (None, ctypes.c_int) for n in (
        "fx_cache_create", "fx_cache_destroy", "fx_cache_set_tables", "fx_cache_scalars", "fx_cache_reserve_sketch",
        "fx_cache_reserve_slots", "fx_cache_probe", "fx_cache_offer", "fx_cache_set_budget", "fx_cache_stage",
        "fx_cache_apply_pending", "fx_cache_age", "fx_cache_lookup", "fx_cache_sketch_estimate",
        "fx_cache_sketch_bump", "fx_cache_sketch_ranked", "fx_cache_lru", "fx_cache_eviction_log",
        "fx_cache_pending", "fx_cache_last_evicted", "fx_cache_set_pending_rows", "fx_cache_set_parallel",
        "fx_cache_advance_tick", "fx_cache_pooled_find", "fx_cache_pooled_touch", "fx_cache_read_slots",
        "fx_cache_pooled_put", "fx_cache_rows", "fx_cache_scalars_device", "fx_cache_capacity", "fx_cache_queue_valid",
        # fused batch step, typed in step.py
        "fx_step_create", "fx_step_destroy", "fx_step_prepare", "fx_step_start", "fx_step_offer", "fx_step_maintain",
        "fx_step_scalars", "fx_step_scalars_device", "fx_step_launches", "fx_step_join")},
    "fx_bag_fingerprint": ([_P, _P, _P, _I32, _P, _I64, _P, _P, _P], ctypes.c_int),
    "fx_store_create": ([ctypes.POINTER(_P), _I32, _I32, _P, _P, _I32, _P, _I32, _U64, _P], ctypes.c_int),
    "fx_store_destroy": ([_P], ctypes.c_int),
    "fx_store_shard_view": ([_P, _I32, _I64, ctypes.POINTER(_P), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                             ctypes.POINTER(_I64), ctypes.POINTER(_I32)], ctypes.c_int),
    "fx_poll_error": ([_P, _P, ctypes.POINTER(_I32), ctypes.POINTER(_I64), _P], ctypes.c_int),
    "fx_comm_init": ([ctypes.POINTER(_P), _I32, _I32, _I64], ctypes.c_int),
    "fx_comm_handle": ([_P, ctypes.c_char_p], ctypes.c_int),
    "fx_comm_connect": ([_P, ctypes.c_char_p], ctypes.c_int),
    "fx_alltoallv": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "fx_comm_recv_buffer": ([_P], _P),
    "fx_comm_recv_counts": ([_P], _P),
    "fx_comm_status": ([_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32)], ctypes.c_int),
    "fx_comm_destroy": ([_P], ctypes.c_int),
}

EXPORTED = []
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name, None)
    if _fn is None:
        continue
    if _args is not None:
        _fn.argtypes = _args
    _fn.restype = _res
    EXPORTED.append(_name)


def check(rc: int, what: str = "") -> None:
    if rc != FX_OK:
        msg = lib.fx_last_error().decode(errors="replace")
        raise _CODE_TO_EXC.get(rc, errors.EmbServeError)(f"{what}: {msg}" if what else msg)


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    if t is None:
        return None
    return int(t.data_ptr())


def idx_type_of(t: torch.Tensor) -> int:
    if t.dtype == torch.int32:
        return FX_IDX_I32
    if t.dtype == torch.int64:
        return FX_IDX_I64
    raise errors.ConfigError(f"indices must be int32 or int64, got {t.dtype}")


def check_out(out: torch.Tensor, rows: int, cols: int, name: str = "out", dtype=torch.float32) -> None:
    """A caller-supplied output buffer must be a CUDA tensor of `dtype`, unit
    column stride and at least [rows, cols] (K4 writes rows*cols elements)."""
    if not out.is_cuda or out.dtype != dtype:
        raise errors.ConfigError(f"{name} must be a CUDA {dtype} tensor, got {out.dtype} on {out.device}")
    if out.dim() != 2 or out.shape[0] < rows or out.shape[1] < cols or (out.shape[1] > 1 and out.stride(1) != 1):
        raise errors.ConfigError(f"{name} must be a row-major [>= {rows}, >= {cols}] tensor, got shape "
                                 f"{tuple(out.shape)} strides {tuple(out.stride())}")


def vec_ok(*ptrs_and_strides) -> bool:
    """True when every (pointer, element-stride) pair is 16-byte aligned for
    4-byte elements (the vector / bulk-copy K4 kernels' requirement)."""
    for p, st in ptrs_and_strides:
        if int(p) % 16 or int(st) % 4:
            return False
    return True


def require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise errors.ConfigError(f"{name} must be a CUDA tensor")


class Status:
    """Device-side first-error word: err[0] = min bad CSR position (INT64_MAX
    when clean), code[0] = FX_E_* of the last violation (0 when clean)."""

    def __init__(self, device):
        self.err = torch.full((1,), INT64_MAX, dtype=torch.int64, device=device)
        self.code = torch.zeros((1,), dtype=torch.int32, device=device)

    def reset(self):
        self.err.fill_(INT64_MAX)
        self.code.zero_()

    def read(self):
        """[sync] -> (code, position)."""
        code = int(self.code.item())
        pos = int(self.err.item())
        return code, pos


def bounds_report():
    """FX_BOUNDS builds (libflexemb_chk.so): {violations, base, index, length}
    of the first out-of-range device subscript on the current device; None
    for a normal build."""
    out = (_I64 * 4)()
    rc = lib.fx_bounds_report(out)
    if rc < 0:
        raise RuntimeError("fx_bounds_report: " + lib.fx_last_error().decode())
    if rc == 0:
        return None
    return {"violations": out[0], "base": out[1], "index": out[2], "length": out[3]}
