"""Sharded lookup on >= 2 GPUs (torchrun, NCCL) vs the CPU oracle."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("exchange", ["nccl", "p2p", "p2p-pipe", "p2p-host"])
@pytest.mark.parametrize("mode", ["tablewise", "rowwise"])
def test_sharded_multi_gpu(mode, exchange):
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "scripts", "sharded_check.py"),
           mode, exchange]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"SHARDED {mode} {exchange}" in r.stdout


def test_sharded_hybrid_replicated_p2p():
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", "29572", os.path.join(ROOT, "scripts", "sharded_check.py"),
           "tablewise", "p2phybrid"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SHARDED tablewise p2phybrid" in r.stdout


def test_sharded_rowwise_f32_partials():
    """f32 partials (the reference's PartialResult format): within tolerance of flat."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", "29573", os.path.join(ROOT, "scripts", "sharded_check.py"),
           "rowwise", "p2pf32"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SHARDED rowwise p2pf32" in r.stdout


@pytest.mark.parametrize("mode,exchange", [("rowwise", "p2pthr"), ("rowwise", "p2pthr32"),
                                           ("rowwise", "p2pthr32-pipe"), ("tablewise", "p2pthr")])
def test_sharded_planned_raw_fetch(mode, exchange):
    """Reference plan (threshold 2) in row-wise mode: singleton (bag, rank)
    groups raw-fetched over NVLink by the requester, larger ones pushed down.
    Per-bag counters equal the reference plan's; with f32 partials the result
    is bit-identical to the reference's hierarchical combine_partials."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", "29574", os.path.join(ROOT, "scripts", "sharded_check.py"),
           mode, exchange]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"SHARDED {mode} {exchange}" in r.stdout
    assert "counter_mismatches=0" in r.stdout and "non_bit_exact_vs_reference_combine=0" in r.stdout


@pytest.mark.parametrize("args", [["2"], ["none"], ["2", "pooled"]])
def test_sharded_ranker_with_per_gpu_caches(args):
    """Ranker pipeline on every rank with its own GPU cache over a sharded
    store (ShardedRanker): metrics, counters, LRU order and eviction log
    equal the canonical-order oracle batch by batch; vectors within the
    reference tolerance."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", "29575",
           os.path.join(ROOT, "scripts", "sharded_ranker_check.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SHARDED_RANKER" in r.stdout and "lru_mismatch_batches=0" in r.stdout


def test_peer_alltoallv_matches_nccl():
    """fx_comm / fx_alltoallv vs NCCL all_to_all_single."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", "29573", os.path.join(ROOT, "scripts", "comm_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"COMM OK world={w}" in r.stdout


@pytest.mark.parametrize("mode,exchange", [("tablewise", "p2p"), ("rowwise", "p2p"), ("rowwise", "p2pthr"),
                                           ("tablewise", "p2p-pipe")])
def test_sharded_two_ranks_folded_on_one_gpu(mode, exchange):
    """The fused exchange with 2 ranks on ONE GPU (FX_FOLD_DEVICES=1): every
    owner / requester store goes through a same-device CUDA-IPC mapping of the
    other process's buffers, the peer barrier through IPC-mapped flags; the
    protocol and the reference plan (threshold 2: raw fetch of the other
    rank's rows) checked against the oracle on a single-GPU box."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29574", os.path.join(ROOT, "scripts", "sharded_check.py"),
           mode, exchange]
    env = dict(os.environ, FX_FOLD_DEVICES="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"SHARDED {mode} {exchange}" in r.stdout and "world=2" in r.stdout


@pytest.mark.parametrize("args", [["2"], ["none"]])
def test_sharded_ranker_folded_on_one_gpu(args):
    """ShardedRanker (per-rank GPU caches over a sharded store) with 2 ranks
    folded onto one GPU: per-batch metrics, counters, LRU order, eviction log
    vs the canonical-order oracle of the same topology."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29576",
           os.path.join(ROOT, "scripts", "sharded_ranker_check.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ, FX_FOLD_DEVICES="1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "SHARDED_RANKER" in r.stdout and "lru_mismatch_batches=0" in r.stdout


def test_sharded_bigcheck_cfg4r_folded_on_one_gpu():
    """cfg4r-sized table-wise exchange (100 tables x 1M rows x 128, B=4096,
    L=20) with 2 ranks folded onto one GPU: sampled bags bit-exact vs the
    flat f64 oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29577",
           os.path.join(ROOT, "scripts", "sharded_bigcheck.py"), "cfg4r", "--bags", "500", "--steps", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ, FX_FOLD_DEVICES="1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert '"max_non_bit_exact": 0' in r.stdout and '"counter_mismatches": 0' in r.stdout
