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
