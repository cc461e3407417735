"""Parity at BASELINE.json sizes: full batches pooled on the GPU; the CPU
oracle checks a random sample of bags bit-exactly (f64 sequential sums,
one rounding), and a size-independent property covers every bag:
linearity — the sum over all bags of their pooled f64 partials equals the
f64 sum of all gathered rows (K4 FX_OUT_F64_PARTIAL vs a second, independent
gather path through fx_gather_rows)."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_12794_b200 as P
    return P


@pytest.mark.parametrize("cfg_key,alpha", [("cfg2", None), ("cfg2", 0.0), ("cfg1", None)])
def test_full_batch_sampled_bags_bit_exact(P, cfg_key, alpha):
    from paper_2410_12794_b200.workload import CONFIGS, DlrmBatchGen
    cfg = CONFIGS[cfg_key]
    rows, D, B = cfg["table_rows"], cfg["dim"], cfg["batch"]
    dep = P.init_store([P.TableMeta(t, n, D) for t, n in enumerate(rows)],
                       [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(rows)], seed=0)
    hb = DlrmBatchGen(rows, cfg["alpha"] if alpha is None else alpha, B, cfg["pooling"], seed=5).next()
    eng = P.LookupEngine(dep)
    out = eng.pool(P.CsrBatch(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(),
                              hb.feature_tables, hb.feature_ops, B)).cpu().numpy()
    rng = np.random.default_rng(0)
    F = len(rows)
    for b in rng.choice(F * B, size=1500, replace=False):
        f, s = divmod(int(b), B)
        ix = hb.indices[hb.offsets[b]:hb.offsets[b + 1]]
        ref = O.pool_flat(O.rows_of(0, f, D, ix), "sum")
        assert ref.tobytes() == out[s, f * D:(f + 1) * D].tobytes(), (f, s)
    del dep, eng


def test_full_batch_linearity_all_bags(P):
    """Sum over bags of f64 partial pools == f64 sum of all gathered rows."""
    from paper_2410_12794_b200 import _lib
    from paper_2410_12794_b200.store import pool_csr_device
    from paper_2410_12794_b200.workload import CONFIGS, DlrmBatchGen
    cfg = CONFIGS["cfg2"]
    rows, D, B = cfg["table_rows"], cfg["dim"], cfg["batch"]
    hb = DlrmBatchGen(rows, cfg["alpha"], B, cfg["pooling"], seed=9).next()
    for f in (2, 11, 15):  # the three largest tables
        t = P.store.table_block_device(0, f, D, 0, rows[f])
        offs = torch.from_numpy(hb.offsets[f * B:(f + 1) * B + 1] - hb.offsets[f * B]).cuda()
        ix = torch.from_numpy(hb.indices[hb.offsets[f * B]:hb.offsets[(f + 1) * B]]).cuda()
        part = pool_csr_device(t, 0, rows[f], ix, offs, "sum", partial=True)
        gathered = torch.empty((ix.numel(), D), dtype=torch.float32, device="cuda")
        st = _lib.Status(torch.device("cuda"))
        _lib.check(_lib.lib.fx_gather_rows(t.data_ptr(), D, 0, rows[f], D, ix.data_ptr(), _lib.FX_IDX_I32,
                                           ix.numel(), gathered.data_ptr(), st.err.data_ptr(), st.code.data_ptr(),
                                           _lib.stream_ptr()))
        a = part.sum(0)
        b_ = gathered.double().sum(0)
        assert torch.allclose(a, b_, rtol=1e-12, atol=1e-9)
        # and the raw gather itself is bit-exact against the PRF for a sample
        sel = np.random.default_rng(f).choice(ix.numel(), size=500, replace=False)
        assert gathered[torch.from_numpy(sel).cuda()].cpu().numpy().tobytes() == \
            O.rows_of(0, f, D, ix.cpu().numpy()[sel]).tobytes()
        del t
