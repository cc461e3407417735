"""Host-side control logic of the mirror package (no GPU needed)."""

import json
import math
import os

import numpy as np
import pytest

from paper_2410_12794_b200 import wire
from paper_2410_12794_b200.errors import ConfigError, EmbServeError, LookupValidationError
from paper_2410_12794_b200.pooling import PlanMode, plan_hierarchical
from paper_2410_12794_b200.routing import build_routing
from paper_2410_12794_b200.store import ShardSpec, TableMeta, validate_placement


def test_placement_errors_match_reference_messages():
    m = {0: TableMeta(0, 4, 2)}
    with pytest.raises(ConfigError, match=r"overlap at row 1"):
        validate_placement(m, [ShardSpec(0, 0, 2, 0), ShardSpec(0, 1, 4, 1)])
    with pytest.raises(ConfigError, match=r"gap \[2,3\)"):
        validate_placement(m, [ShardSpec(0, 0, 2, 0), ShardSpec(0, 3, 4, 1)])
    with pytest.raises(ConfigError, match="beyond"):
        validate_placement(m, [ShardSpec(0, 0, 5, 0)])
    with pytest.raises(ConfigError, match="gap"):
        validate_placement({0: TableMeta(0, 4, 2), 1: TableMeta(1, 4, 2)}, [ShardSpec(0, 0, 4, 0)])
    with pytest.raises(ConfigError):
        TableMeta(0, 0, 4)
    with pytest.raises(ConfigError):
        TableMeta(0, 4, 4, element_width=2)


def test_plan_threshold_semantics():
    plan = plan_hierarchical({(0, 0): 2, (1, 0): 1}, threshold=2)
    assert plan.mode(0, 0) is PlanMode.PUSHDOWN and plan.mode(1, 0) is PlanMode.RAW_FETCH
    with pytest.raises(EmbServeError):
        plan_hierarchical({}, threshold=1)


def test_wire_byte_model():
    assert wire.embedding_payload_bytes(8, 64) == 2048 == 8 * wire.embedding_payload_bytes(1, 64)
    assert wire.partial_response_bytes(64) == 32 + 256 + 8
    assert wire.raw_response_bytes(8, 64) == 32 + 2048
    assert wire.request_bytes(3) == 32 + 24


def test_scalar_resolve_matches_golden(golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "routing.json")))
    for c in cases:
        pl = [ShardSpec(*s) for s in c["placement"]]
        rt = build_routing([TableMeta(0, c["num_rows"], 4)], pl)
        assert [list(e) for e in rt.entries(0)] == [list(e) for e in c["entries"]]
        for i, s in zip(c["idx"][:100], c["servers"][:100]):
            assert rt.resolve(0, i) == s


def test_resolve_comparison_count_logarithmic():
    rng = np.random.default_rng(7)
    for shards in (1, 2, 7, 33, 128):
        bounds = np.linspace(0, 4096, shards + 1).astype(int)
        rt = build_routing([TableMeta(0, 4096, 4)],
                           [ShardSpec(0, int(bounds[i]), int(bounds[i + 1]), i % 4) for i in range(shards)])
        for idx in rng.integers(0, 4096, size=100):
            cnt = [0]
            rt.resolve(0, int(idx), counter=cnt)
            assert cnt[0] <= math.ceil(math.log2(shards)) + 1


def test_resolve_out_of_range_and_unknown_table():
    rt = build_routing([TableMeta(0, 200, 4)], [ShardSpec(0, 0, 100, 0), ShardSpec(0, 100, 200, 1)])
    assert rt.resolve(0, 99) == 0 and rt.resolve(0, 100) == 1
    for bad in (200, -1):
        with pytest.raises(LookupValidationError):
            rt.resolve(0, bad)
    with pytest.raises(LookupValidationError):
        rt.resolve(9, 0)


# names exported by the reference package (embserve/__init__.py:13-28)
REFERENCE_EXPORTS = (
    "AdaptiveCache CachePolicy LoadLevel LoadTracker MemoryModel CapacityError ConfigError EmbServeError "
    "FlowControlError InvariantError LookupValidationError RoutingViolationError TraceParseError PartialResult "
    "PlanMode PoolingOp combine_partials pool_flat Batch Feature LookupRequest RoutingTable build_routing "
    "group_by_server Deployment ServerStore ShardSpec TableMeta init_store Trace WorkloadConfig generate_trace "
    "load_trace save_trace").split()


def test_reference_public_api_is_exported():
    import paper_2410_12794_b200 as P
    missing = [n for n in REFERENCE_EXPORTS if not hasattr(P, n)]
    assert not missing, missing


def test_cache_control_logic_host_side():
    from paper_2410_12794_b200.cache import (CachePolicy, LoadLevel, LoadTracker, MemoryModel,
                                             max_batch_for_cache, target_cache_bytes)
    from paper_2410_12794_b200.errors import CapacityError
    m = MemoryModel(gpu_capacity_bytes=1000, nn_fixed_bytes=200, nn_per_sample_bytes=1)
    assert target_cache_bytes(m, 400) == 400 and target_cache_bytes(m, 800) == 0
    with pytest.raises(CapacityError):
        target_cache_bytes(m, 900)
    assert max_batch_for_cache(m, 400) == 400 and max_batch_for_cache(m, 0) == 800
    with pytest.raises(ConfigError):
        MemoryModel(gpu_capacity_bytes=10, nn_fixed_bytes=20, nn_per_sample_bytes=1)
    tr = LoadTracker(window=4, high_watermark=512, low_watermark=128)
    for _ in range(4):
        lvl = tr.record_batch(600)
    assert lvl is LoadLevel.HIGH
    tr = LoadTracker(window=2, high_watermark=100, low_watermark=10)
    tr.record_batch(500)
    tr.record_batch(50)
    assert tr.record_batch(50) is LoadLevel.NORMAL
    assert LoadTracker(window=4, high_watermark=512, low_watermark=128, stat="max").record_batch(600) is LoadLevel.HIGH
    pm = MemoryModel(gpu_capacity_bytes=10_000, nn_fixed_bytes=1_000, nn_per_sample_bytes=10)
    pol = CachePolicy(model=pm, hysteresis_fraction=0.0)
    assert pol.propose(1_000, LoadLevel.HIGH, windowed_batch=100) <= 1_000
    assert pol.propose(9_000, LoadLevel.LOW, windowed_batch=800) >= 9_000
    assert pol.propose(0, LoadLevel.NORMAL, windowed_batch=100) == 8_000
    pol = CachePolicy(model=pm, hysteresis_fraction=0.05)
    assert pol.propose(7_800, LoadLevel.NORMAL, windowed_batch=100) == 7_800
    assert pol.propose(7_000, LoadLevel.NORMAL, windowed_batch=100) == 8_000
    assert CachePolicy(model=pm, hysteresis_fraction=0.0).propose(5_000, LoadLevel.HIGH, windowed_batch=2_000) == 0
