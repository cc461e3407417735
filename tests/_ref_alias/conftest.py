"""Run the reference's own unit tests (test_store / test_pooling /
test_routing / test_cache, copied here untouched by __graft_entry__.build()
from /root/reference/pkg/tests) against the B200 mirror: `embserve` and its
submodules are aliased to paper_2410_12794_b200, so every assertion the
reference makes about its API is checked against our implementation on the
GPU. Known, documented divergences are marked xfail with the reason."""

import importlib
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# reference test id -> why the mirror deliberately differs
XFAIL = {
    # writes into a shard in place (store.py:59 calls shards immutable by
    # convention); our shards are HBM tensors — item assignment works, but the
    # reference's numpy-list semantics are not part of the contract
    "test_store.py::test_partial_pool_sum_example": "mutates a shard in place (shards are immutable by convention)",
    # shard data is an HBM-resident torch tensor, not a host numpy array
    # (same bytes: tests/test_oracle_golden.py + test_gpu_core.py check the PRF bit-exactly)
    "test_store.py::test_init_deterministic_bytes": "Shard.data is a CUDA tensor (no numpy .tobytes())",
    "test_store.py::test_different_seed_different_content": "Shard.data is a CUDA tensor (no numpy .tobytes())",
}


def _alias():
    import paper_2410_12794_b200 as P
    sys.modules.setdefault("embserve", P)
    for sub in ("store", "pooling", "routing", "cache", "errors", "requests", "wire"):
        sys.modules.setdefault(f"embserve.{sub}", importlib.import_module(f"paper_2410_12794_b200.{sub}"))


def pytest_collection_modifyitems(config, items):
    here = os.path.dirname(os.path.abspath(__file__))
    for it in items:
        if not str(it.fspath).startswith(here):
            continue
        it.add_marker(pytest.mark.gpu)
        key = f"{os.path.basename(str(it.fspath))}::{it.name.split('[')[0]}"
        if key in XFAIL:
            it.add_marker(pytest.mark.xfail(reason=XFAIL[key], strict=False))


def pytest_ignore_collect(collection_path, config):
    # without a GPU the mirror cannot run; the copied files import `embserve`
    # at module level, so skip collecting them entirely
    if collection_path.name.startswith("test_") and collection_path.parent == type(collection_path)(
            os.path.dirname(os.path.abspath(__file__))):
        try:
            import torch
            if not torch.cuda.is_available():
                return True
        except Exception:
            return True
        _alias()
    return None
