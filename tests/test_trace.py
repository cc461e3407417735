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


def test_dlrm_dataset_loader_and_converter(tmp_path):
    """Fast CSR loader for DLRM lookup datasets (indices, offsets, lengths;
    table-major bags) and the dlrm-tensors external trace converter."""
    import torch
    from paper_2410_12794_b200.trace import convert_external_trace, iter_dlrm_batches
    rng = np.random.default_rng(0)
    T, N, B = 3, 10, 4
    lengths = rng.integers(1, 5, (T, N))
    offsets = np.concatenate([[0], np.cumsum(lengths.reshape(-1))])
    indices = rng.integers(0, 1000, int(offsets[-1]))
    path = tmp_path / "day.pt"
    torch.save((torch.from_numpy(indices), torch.from_numpy(offsets), torch.from_numpy(lengths)), path)
    hbs = list(iter_dlrm_batches(str(path), B, ops=("sum", "mean", "sum")))
    assert len(hbs) == N // B
    for k, hb in enumerate(hbs):
        for t in range(T):
            for s in range(B):
                b = t * N + k * B + s
                got = hb.indices[hb.offsets[t * B + s]:hb.offsets[t * B + s + 1]]
                assert list(got) == list(indices[offsets[b]:offsets[b + 1]])
    tr = convert_external_trace(str(path), "dlrm-tensors", batch_size=B, ops=("sum", "mean", "sum"))
    assert len(tr.batches) == 2 and tr.batches[1].lookups[2].features[1].op.value == "mean"
    assert tr.batches[0].lookups[0].features[0].indices == list(indices[offsets[0]:offsets[1]])
    with pytest.raises(NotImplementedError):
        convert_external_trace(str(path), "criteo-raw")


def test_metrics_report_schema_vs_reference(golden_dir):
    """MetricsReport / percentiles reproduce the reference's text and
    canonical machine forms (bench/report.py) byte for byte."""
    import json
    from paper_2410_12794_b200.report import MetricsReport, RunMetrics, percentiles
    g = json.load(open(f"{golden_dir}/report.json"))
    for c, p in zip(g["cases"], g["percentiles"]):
        assert percentiles(c) == p
    rep = MetricsReport(experiment="golden-x", seed=7, backend="virtual", fingerprint="abc123",
                        config={"b": 2, "a": [1, 2]},
                        runs=[RunMetrics(label="r1", makespan=12.5, throughput=3.25, throughput_unit="lookups/tick",
                                         counters={"z": 1, "a": 2},
                                         latency_stages={"net": percentiles([1.0, 2.0, 4.0])}, extras={"note": "x"}),
                              RunMetrics(label="r2", throughput_unit="lookups/tick")],
                        comparison={"speedup": 1.5}, invariants={"ok": True})
    assert rep.to_machine() == g["machine"]
    assert rep.to_text() == g["text"]


def test_numa_cpulist_parser():
    from paper_2410_12794_b200.numa import _parse_cpulist
    assert _parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert _parse_cpulist("") == []
