"""Synthetic inputs: same Zipf semantics as the reference sampler, deterministic."""

import os

import numpy as np

import oracle as O
from paper_2410_12794_b200.workload import DlrmBatchGen, ZipfSampler


def test_zipf_matches_oracle_and_golden(golden_dir):
    z = np.load(os.path.join(golden_dir, "zipf.npz"))
    for i in range(4):
        n, a, seed, k = z[f"meta{i}"]
        got = ZipfSampler(int(n), float(a)).sample(np.random.default_rng(int(seed)), int(k))
        assert np.array_equal(got, z[f"s{i}"])


def test_dlrm_gen_deterministic_and_table_major():
    g1 = DlrmBatchGen((1000, 50, 7), 1.05, 16, (1, 5), seed=3)
    g2 = DlrmBatchGen((1000, 50, 7), 1.05, 16, (1, 5), seed=3)
    a, b = g1.next(), g2.next()
    assert np.array_equal(a.indices, b.indices) and np.array_equal(a.offsets, b.offsets)
    assert a.offsets.size == 3 * 16 + 1
    for f, n in enumerate((1000, 50, 7)):
        seg = a.indices[a.offsets[f * 16]:a.offsets[(f + 1) * 16]]
        assert seg.min() >= 0 and seg.max() < n
    lens = np.diff(a.offsets)
    assert lens.min() >= 1 and lens.max() <= 5


def test_dlrm_gen_uniforms_follow_zipf_inverse_cdf():
    g = DlrmBatchGen((100_000,), 1.05, 64, 20, seed=0)
    hb = g.next()
    rng = np.random.default_rng(0)
    u = rng.random(64 * 20)
    ref = O.ZipfSampler(100_000, 1.05).sample(np.random.default_rng(0), 64 * 20)
    assert np.array_equal(np.minimum(ref, 99_999), hb.indices)


def test_permutation_is_bijective():
    g = DlrmBatchGen((1009,), 1.0, 4, 2, permute=True)
    rows = np.arange(1009, dtype=np.int32)
    p = g._perm(rows, 1009, 0)
    assert np.array_equal(np.sort(p), rows)
