"""GPU parity: libflexemb kernels vs the CPU oracle and the reference's golden
vectors. Integer/byte/index outputs must be bit-exact; pooled f32 outputs
must satisfy |a-b| <= max(1e-6, 1e-5|ref|) (ranker.py:487-491) and are
additionally expected bit-identical to the flat f64 oracle."""

import json
import os

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

REL, ABS = 1e-5, 1e-6  # north-star tolerance, BASELINE.md


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_12794_b200 as P
    return P


# ---------------------------------------------------------------- K0 store

def test_table_block_bit_exact_vs_golden(P, golden_dir):
    z = np.load(os.path.join(golden_dir, "prf.npz"))
    i = 0
    while f"case{i}" in z:
        seed, t, d, s, e = (int(v) for v in z[f"case{i}"])
        assert P.table_block(seed, t, d, s, e).tobytes() == z[f"block{i}"].tobytes(), i
        i += 1
    for k, r in enumerate((0, 1, 77, 99_999)):
        assert P.row_values(3, 2, r, 64).tobytes() == z["rowv"][k].tobytes()


def test_table_init_large_table_sampled_rows(P):
    # 10M-row table, D=128: sampled rows bit-exact vs the oracle PRF
    t = P.store.table_block_device(0, 7, 128, 0, 10_000_000)
    rows = np.array([0, 1, 4_999_999, 9_999_999, 123_457])
    got = t[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert got.tobytes() == O.rows_of(0, 7, 128, rows).tobytes()
    assert float(t.max()) <= 1.0 and float(t.min()) >= -1.0
    del t


def test_store_determinism_and_lookup_rows(P):
    dep = P.init_store([P.TableMeta(0, 8, 2)], [P.ShardSpec(0, 0, 8, 0)], seed=7)
    dep2 = P.init_store([P.TableMeta(0, 8, 2)], [P.ShardSpec(0, 0, 8, 0)], seed=7)
    s = dep.servers[0]
    assert s.shards(0)[0].data.cpu().numpy().tobytes() == dep2.servers[0].shards(0)[0].data.cpu().numpy().tobytes()
    rows = s.lookup_rows(0, [0, 0, 3])
    assert rows.shape == (3, 2) and np.array_equal(rows[0], rows[1]) and not np.array_equal(rows[0], rows[2])
    assert s.lookup_rows(0, []).shape == (0, 2)
    fwd = s.lookup_rows(0, [1, 5, 2])
    assert np.array_equal(fwd, O.rows_of(7, 0, 2, [1, 5, 2]))


def test_unhosted_row_is_routing_violation(P):
    dep = P.init_store([P.TableMeta(0, 8, 2)], [P.ShardSpec(0, 0, 4, 0), P.ShardSpec(0, 4, 8, 1)], seed=0)
    with pytest.raises(P.RoutingViolationError):
        dep.servers[0].lookup_rows(0, [5])
    with pytest.raises(P.RoutingViolationError):
        dep.servers[1].partial_pool(0, [1, 6], P.PoolingOp.SUM)


def test_partial_pool_bit_exact_vs_golden(P, golden_dir):
    z = np.load(os.path.join(golden_dir, "pool.npz"))
    for k in range(int(z["n_pp"][0])):
        seed, rows, dim = (int(v) for v in z[f"pp{k}_meta"])
        dep = P.init_store([P.TableMeta(0, rows, dim)], [P.ShardSpec(0, 0, rows, 0)], seed=seed)
        idx = z[f"pp{k}_idx"].tolist()
        pr = dep.servers[0].partial_pool(0, idx, P.PoolingOp.SUM)
        assert pr.count == len(idx)
        assert pr.vector.tobytes() == z[f"pp{k}_vec"].tobytes(), (k, dim)
        assert dep.servers[0].lookup_rows(0, idx).tobytes() == z[f"pp{k}_raw"].tobytes()
    with pytest.raises(P.EmbServeError, match="empty partial pool"):
        dep.servers[0].partial_pool(0, [], P.PoolingOp.SUM)


def test_multi_shard_server_partial_pool(P):
    # one server hosting two shards of a table: input-order sum across shards
    dep = P.init_store([P.TableMeta(0, 100, 16)], [P.ShardSpec(0, 0, 40, 0), P.ShardSpec(0, 40, 70, 1),
                                                    P.ShardSpec(0, 70, 100, 0)], seed=3)
    idx = [75, 1, 99, 39, 80, 0]
    pr = dep.servers[0].partial_pool(0, idx, P.PoolingOp.SUM)
    assert pr.vector.tobytes() == O.seq_sum_f64(O.rows_of(3, 0, 16, idx)).astype(np.float32).tobytes()
    assert dep.servers[0].lookup_rows(0, idx).tobytes() == O.rows_of(3, 0, 16, idx).tobytes()


# ---------------------------------------------------------------- K4/K5 pooling

def test_pool_flat_and_combine_vs_golden(P, golden_dir):
    z = np.load(os.path.join(golden_dir, "pool.npz"))
    for k in range(int(z["n_c"][0])):
        rows = z[f"c{k}_rows"]
        owners = z[f"c{k}_owner"]
        pushed = set(int(g) for g in z[f"c{k}_pushed"])
        op = P.PoolingOp.SUM if int(z[f"c{k}_op"][0]) == 0 else P.PoolingOp.MEAN
        partials, raw_pos = [], []
        for g in np.unique(owners):
            mem = np.nonzero(owners == g)[0]
            if int(g) in pushed:
                vec = P.pooling.sum_rows_f64(rows[mem]).astype(np.float32)
                partials.append(P.PartialResult(vector=vec, count=len(mem), source=int(g)))
            else:
                raw_pos.extend(mem.tolist())
        raw = [rows[i] for i in sorted(raw_pos)]
        got = P.combine_partials(partials, raw, op)
        assert got.tobytes() == z[f"c{k}_comb"].tobytes(), k
        assert P.pool_flat(list(rows), op).tobytes() == z[f"c{k}_flat"].tobytes(), k


def test_combine_examples(P):
    pr = P.PartialResult(vector=np.array([4, 6], np.float32), count=2, source=0)
    raw = [np.array([5, 5], np.float32)]
    assert np.allclose(P.combine_partials([pr], raw, P.PoolingOp.SUM), [9, 11])
    assert np.allclose(P.combine_partials([pr], raw, P.PoolingOp.MEAN), [3.0, 11.0 / 3.0])
    with pytest.raises(P.EmbServeError):
        P.combine_partials([], [], P.PoolingOp.SUM)
    with pytest.raises(P.EmbServeError, match="dim mismatch"):
        P.pool_flat([np.ones(2, np.float32), np.ones(3, np.float32)], P.PoolingOp.SUM)


def _engine_batch(P, tables, dims, B, pooling, alpha, seed, ops=None, idx_dtype=np.int32):
    from paper_2410_12794_b200.workload import DlrmBatchGen
    metas = [P.TableMeta(t, n, d) for t, (n, d) in enumerate(zip(tables, dims))]
    placement = [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(tables)]
    dep = P.init_store(metas, placement, seed=0)
    g = DlrmBatchGen(tables, alpha, B, pooling, seed=seed, ops=ops)
    hb = g.next()
    return dep, hb


def _oracle_pool(hb, dims):
    bb = O.BagBatch(hb.offsets, hb.indices.astype(np.int64),
                    np.repeat(np.array(hb.feature_tables), hb.batch_size),
                    [op for op in hb.feature_ops for _ in range(hb.batch_size)],
                    np.tile(np.arange(hb.batch_size), len(hb.feature_tables)),
                    np.repeat(np.arange(len(hb.feature_tables)), hb.batch_size), hb.batch_size)
    return O.flat_pool_batch(0, dict(enumerate(dims)), bb)


@pytest.mark.parametrize("dim,B,L", [(64, 512, 20), (128, 256, (1, 40)), (32, 64, 7), (256, 64, (1, 9)),
                                     (12, 64, 5), (7, 32, (1, 33)), (520, 16, 3), (1, 16, 4)])
def test_engine_pool_vs_oracle(P, dim, B, L):
    tables = (1000, 37, 5000)
    dims = (dim,) * 3
    ops = ("sum", "mean", "sum")
    dep, hb = _engine_batch(P, tables, dims, B, L, 1.05, seed=dim, ops=ops)
    eng = P.LookupEngine(dep)
    batch = P.CsrBatch(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(),
                       hb.feature_tables, hb.feature_ops, hb.batch_size)
    out = eng.pool(batch).cpu().numpy()
    ref = _oracle_pool(hb, dims)
    F = len(tables)
    exact = 0
    for f in range(F):
        for s in range(B):
            r = ref[f * B + s]
            g = out[s, f * dim:(f + 1) * dim]
            assert O.within_tolerance(r, g)
            exact += r.tobytes() == g.tobytes()
    assert exact == F * B  # f64 sequential accumulation: bit-identical to the flat oracle


@pytest.mark.parametrize("dim", [64, 128, 12])
def test_pool_many_requests_one_launch(P, dim):
    """LookupEngine.pool_many: many independent requests in ONE K4 launch,
    bit-identical to pooling each request on its own (and to the oracle)."""
    from paper_2410_12794_b200.workload import DlrmBatchGen
    tables = (1000, 37, 5000)
    dims = (dim,) * 3
    ops = ("sum", "mean", "sum")
    dep = P.init_store([P.TableMeta(t, n, dim) for t, n in enumerate(tables)],
                       [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(tables)], seed=0)
    eng = P.LookupEngine(dep)
    reqs, hbs = [], []
    for r in range(9):
        hb = DlrmBatchGen(tables, 1.05, 8 + 7 * r, (0, 12), seed=50 + r, ops=ops).next()
        hbs.append(hb)
        reqs.append(P.CsrBatch(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(),
                               hb.feature_tables, hb.feature_ops, hb.batch_size))
    outs = eng.pool_many(reqs)
    for hb, req, o in zip(hbs, reqs, outs):
        single = eng.pool(req).cpu().numpy()
        assert o.cpu().numpy().tobytes() == single.tobytes()
        ref = _oracle_pool(hb, dims)
        B = hb.batch_size
        for f in range(3):
            for s in range(B):
                b = f * B + s
                if hb.offsets[b + 1] > hb.offsets[b]:  # empty bags pool to 0 (no reference value)
                    assert ref[b].tobytes() == single[s, f * dim:(f + 1) * dim].tobytes()
    bad = reqs[4].indices.clone()
    bad[3] = 10 ** 6
    reqs[4] = P.CsrBatch(bad, reqs[4].offsets, reqs[4].feature_tables, reqs[4].feature_ops, reqs[4].batch_size)
    with pytest.raises(P.LookupValidationError, match=r"request 4, lookup"):
        eng.pool_many(reqs)


def test_engine_mixed_dims_and_int64(P):
    tables, dims = (300, 500), (16, 64)
    dep, hb = _engine_batch(P, tables, dims, 32, (1, 6), 0.8, seed=1)
    eng = P.LookupEngine(dep)
    batch = P.CsrBatch(torch.from_numpy(hb.indices.astype(np.int64)).cuda(), torch.from_numpy(hb.offsets).cuda(),
                       hb.feature_tables, hb.feature_ops, hb.batch_size)
    out = eng.pool(batch).cpu().numpy()
    ref = _oracle_pool(hb, dims)
    for s in range(32):
        assert out[s, :16].tobytes() == ref[s].tobytes()
        assert out[s, 16:].tobytes() == ref[32 + s].tobytes()


def test_engine_validation_error_message(P):
    dep, hb = _engine_batch(P, (100, 50), (8, 8), 4, 3, 1.0, seed=2)
    idx = hb.indices.copy()
    # lookup 2, feature 1 gets an out-of-range index; lookup 3 feature 0 too (later in sm order)
    idx[hb.offsets[1 * 4 + 2] + 1] = 50
    idx[hb.offsets[0 * 4 + 3]] = 1000
    eng = P.LookupEngine(dep)
    batch = P.CsrBatch(torch.from_numpy(idx).cuda(), torch.from_numpy(hb.offsets).cuda(),
                       hb.feature_tables, hb.feature_ops, 4)
    with pytest.raises(P.LookupValidationError, match=r"batch 0, lookup 2: index 50 out of range \[0,50\) for table 1"):
        eng.pool(batch)


def test_empty_bags_pool_to_zero(P):
    dep = P.init_store([P.TableMeta(0, 10, 8)], [P.ShardSpec(0, 0, 10, 0)], seed=0)
    eng = P.LookupEngine(dep)
    offs = torch.tensor([0, 0, 2, 2], dtype=torch.int64).cuda()
    idx = torch.tensor([3, 4], dtype=torch.int32).cuda()
    out = eng.pool(P.CsrBatch(idx, offs, (0,), ("mean",), 3)).cpu().numpy()
    assert np.all(out[0] == 0) and np.all(out[2] == 0)
    assert out[1].tobytes() == O.pool_flat(O.rows_of(0, 0, 8, [3, 4]), "mean").tobytes()


# ---------------------------------------------------------------- K1 routing

def test_resolve_many_and_group_by_server_vs_golden(P, golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "routing.json")))
    for c in cases:
        rt = P.build_routing([P.TableMeta(0, c["num_rows"], 4)], [P.ShardSpec(*s) for s in c["placement"]])
        assert rt.resolve_many(0, c["idx"]).tolist() == c["servers"]
        groups = P.group_by_server(rt, P.LookupRequest([P.Feature(0, P.PoolingOp.SUM, c["feature"])]))
        assert [[g.server_id, g.items[0].indices, g.items[0].positions] for g in groups] == c["groups"]


def test_routing_errors(P):
    rt = P.build_routing([P.TableMeta(0, 200, 4)], [P.ShardSpec(0, 0, 100, 0), P.ShardSpec(0, 100, 200, 1)])
    with pytest.raises(P.LookupValidationError):
        rt.resolve_many(0, [0, 200])
    with pytest.raises(P.LookupValidationError, match=r"table 0"):
        P.group_by_server(rt, P.LookupRequest([P.Feature(0, P.PoolingOp.SUM, [5, 999])]))
    groups = P.group_by_server(rt, P.LookupRequest([P.Feature(0, P.PoolingOp.SUM, [90, 10, 50])]))
    assert groups[0].items[0].indices == [90, 10, 50]


def test_bucket_stable_per_destination(P):
    from paper_2410_12794_b200 import _lib
    rng = np.random.default_rng(0)
    n_bags, n_dest = 300, 5
    lens = rng.integers(0, 30, size=n_bags)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    dest = rng.integers(0, n_dest, size=offs[-1]).astype(np.int32)
    d_dest, d_offs = torch.from_numpy(dest).cuda(), torch.from_numpy(offs).cuda()
    perm = torch.empty(offs[-1], dtype=torch.int64, device="cuda")
    dc = torch.empty(n_dest, dtype=torch.int64, device="cuda")
    bc = torch.empty(n_dest * n_bags, dtype=torch.int32, device="cuda")
    import ctypes
    ws_bytes = ctypes.c_size_t(0)
    _lib.check(_lib.lib.fx_bucket(d_dest.data_ptr(), int(offs[-1]), d_offs.data_ptr(), n_bags, n_dest,
                                  perm.data_ptr(), dc.data_ptr(), bc.data_ptr(), None, ctypes.byref(ws_bytes), None))
    ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib.fx_bucket(d_dest.data_ptr(), int(offs[-1]), d_offs.data_ptr(), n_bags, n_dest,
                                  perm.data_ptr(), dc.data_ptr(), bc.data_ptr(), ws.data_ptr(),
                                  ctypes.byref(ws_bytes), _lib.stream_ptr()))
    ref_perm = np.argsort(dest, kind="stable")
    assert np.array_equal(perm.cpu().numpy(), ref_perm)
    assert np.array_equal(dc.cpu().numpy(), np.bincount(dest, minlength=n_dest))
    bag_of = np.repeat(np.arange(n_bags), lens)
    ref_bc = np.zeros((n_dest, n_bags), np.int64)
    np.add.at(ref_bc, (dest, bag_of), 1)
    assert np.array_equal(bc.cpu().numpy().reshape(n_dest, n_bags), ref_bc)


# ---------------------------------------------------------------- K2 dedup

def test_dedup_bit_exact_vs_numpy_unique(P):
    from paper_2410_12794_b200.dedup import dedup_csr
    from paper_2410_12794_b200.workload import DlrmBatchGen
    g = DlrmBatchGen((100_000,) * 8, 1.05, 512, 20, seed=0)
    hb = g.next()
    B, F = 512, 8
    idx = torch.from_numpy(hb.indices).cuda()
    offs = torch.from_numpy(hb.offsets).cuda()
    bag_table = torch.arange(F, dtype=torch.int32).repeat_interleave(B).cuda()
    res = dedup_csr(bag_table, idx, offs, B, F)
    keys = O.make_keys(np.repeat(np.arange(F), np.diff(hb.offsets).reshape(F, B).sum(1)), hb.indices)
    u, inv, cnt = O.dedup_keys(keys)
    got_u = res.uniq.cpu().numpy()
    assert got_u.size == u.size
    order = np.argsort(got_u)
    assert np.array_equal(got_u[order], u)               # unique set
    assert np.array_equal(res.mult.cpu().numpy()[order], cnt)   # multiplicities
    ginv = res.inverse.cpu().numpy()
    assert np.array_equal(got_u[ginv], keys)              # inverse map
    # first-occurrence order: ordinals strictly increasing
    fo = res.first_ord.cpu().numpy()
    assert np.all(np.diff(fo) > 0)


def test_pool_mixed_dims_unaligned_columns_and_out_checks(P):
    """Mixed dims (30, 128): the D=128 feature's output column starts 120 B
    into a 632-B row; K4 must take the scalar path there (a 16-B vector
    store would fault) and still match the flat oracle. Bad `out` buffers are
    rejected before any launch."""
    from paper_2410_12794_b200.engine import CsrBatch, LookupEngine
    from paper_2410_12794_b200.workload import DlrmBatchGen
    rows, dims, B = (5000, 7000), (30, 128), 40
    metas = [P.TableMeta(t, n, d) for t, (n, d) in enumerate(zip(rows, dims))]
    dep = P.init_store(metas, [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(rows)], 0)
    hb = DlrmBatchGen(rows, 1.0, B, (1, 9), seed=8).next()
    eng = LookupEngine(dep)
    batch = CsrBatch(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(), hb.feature_tables,
                     hb.feature_ops, B)
    out = eng.pool(batch).cpu().numpy()
    col = 0
    for f, d in enumerate(dims):
        for s in range(B):
            b = f * B + s
            ref = O.pool_flat(O.rows_of(0, f, d, hb.indices[hb.offsets[b]:hb.offsets[b + 1]]), "sum")
            assert ref.tobytes() == out[s, col:col + d].tobytes()
        col += d
    with pytest.raises(P.ConfigError):
        eng.pool(batch, out=torch.empty((B, 100), dtype=torch.float32, device="cuda"))
    with pytest.raises(P.ConfigError):
        eng.pool(batch, out=torch.empty((B, 158), dtype=torch.float64, device="cuda"))
    # an output view at a 4-byte offset (unaligned): scalar path, same values
    big = torch.empty((B, 159), dtype=torch.float32, device="cuda")
    got = eng.pool(batch, out=big[:, 1:]).cpu().numpy()
    assert np.array_equal(got, out)


def test_host_stream_reports_the_failing_batch(P):
    """HostLookup.stream: a bad index in the 3rd of 5 batches raises the
    reference's message for THAT batch when it is yielded (per-slot status)."""
    from paper_2410_12794_b200.engine import CsrBatch, HostLookup, LookupEngine
    from paper_2410_12794_b200.workload import DlrmBatchGen
    rows, D, B = (3000, 4000), 32, 16
    dep = P.init_store([P.TableMeta(t, n, D) for t, n in enumerate(rows)],
                       [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(rows)], 0)
    gen = DlrmBatchGen(rows, 1.0, B, (2, 6), seed=4)
    hbs = [gen.next() for _ in range(5)]
    bad = hbs[2].indices.copy()
    b = 1 * B + 5
    bad[hbs[2].offsets[b]] = 4000 + 3
    batches = []
    for i, hb in enumerate(hbs):
        idx = bad if i == 2 else hb.indices
        batches.append(CsrBatch(torch.from_numpy(idx).pin_memory(), torch.from_numpy(hb.offsets).pin_memory(),
                                hb.feature_tables, hb.feature_ops, B))
    hl = HostLookup(LookupEngine(dep))
    got = []
    with pytest.raises(P.LookupValidationError, match="batch 2, lookup 5: index 4003 out of range"):
        for out in hl.stream(batches, depth=3):
            got.append(out.clone())
    assert len(got) == 2


@pytest.mark.parametrize("row_begin,ld,partial", [(0, 128, False), (1000, 160, False), (0, 132, True)])
def test_pool_strided_shard_vs_oracle(P, row_begin, ld, partial):
    """K4 on a shard whose rows are ld >= dim floats apart and whose first row
    is a global row != 0 (the bulk / gather4 copies address rows by stride)."""
    from paper_2410_12794_b200.store import pool_csr_device
    g = torch.Generator().manual_seed(ld)
    n = 3000
    base = torch.randn(n, ld, generator=g)
    tab = base[:, :128].cuda()  # contiguous copy, then re-stride below
    big = torch.zeros(n, ld, device="cuda")
    big[:, :128] = tab
    view = big[:, :128]
    rng = np.random.default_rng(ld)
    lens = rng.integers(0, 41, size=700)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = (rng.integers(0, n, size=int(offs[-1])) + row_begin).astype(np.int64)
    out = pool_csr_device(view, row_begin, row_begin + n, torch.from_numpy(idx).cuda(), torch.from_numpy(offs).cuda(),
                          "sum", partial=partial).cpu().numpy()
    host = base[:, :128].numpy()
    for b in range(len(lens)):
        if lens[b] == 0:
            continue
        rows = host[idx[offs[b]:offs[b + 1]] - row_begin]
        ref = O.seq_sum_f64(rows)
        if partial:
            assert out[b].tobytes() == ref.tobytes(), b
        else:
            assert out[b].tobytes() == ref.astype(np.float32).tobytes(), b
