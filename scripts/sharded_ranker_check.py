"""torchrun --nproc-per-node N scripts/sharded_ranker_check.py [threshold|none] [pooled]
Every rank runs the Ranker pipeline with its own GPU cache over a store
row/table-sharded across the ranks (ShardedRanker) and is checked, batch by
batch, against the canonical-order CPU oracle of the same topology (servers
= ranks): per-batch metrics, per-bag counters, cache LRU order, eviction log
and pooled vectors (tolerance + bit-exact vs flat)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2410_12794_b200 import cache as C  # noqa: E402
from paper_2410_12794_b200.ranker import RankerParams  # noqa: E402
from paper_2410_12794_b200.sharded import rowwise_placement, tablewise_placement  # noqa: E402
from paper_2410_12794_b200.sharded_ranker import ShardedRanker  # noqa: E402
from paper_2410_12794_b200.store import ShardSpec, TableMeta  # noqa: E402
from paper_2410_12794_b200.workload import DlrmBatchGen  # noqa: E402


def main():
    thr = None if (len(sys.argv) < 2 or sys.argv[1] == "none") else int(sys.argv[1])
    pooled = len(sys.argv) > 2 and sys.argv[2] == "pooled"
    # FX_FOLD_DEVICES=1: ranks folded onto the visible GPUs (one-GPU box: every
    # rank on cuda:0, exchange through same-device IPC mappings, gloo control)
    fold = os.environ.get("FX_FOLD_DEVICES") == "1"
    local = int(os.environ["LOCAL_RANK"]) % (torch.cuda.device_count() if fold else 1 << 30)
    torch.cuda.set_device(local)
    if fold:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    rows = (3000, 120, 2500, 40, 900, 7)
    ops = ("sum", "mean", "sum", "sum", "mean", "sum")
    D, B = 32, 48
    metas = [TableMeta(t, n, D) for t, n in enumerate(rows)]
    # tables 0, 2 row-wise over all ranks, the rest table-wise
    rw = [sp for sp in rowwise_placement(rows, world) if sp.table_id in (0, 2)]
    tw_tabs = [1, 3, 4, 5]
    tw = [ShardSpec(tw_tabs[s.table_id], s.start, s.end, s.server_id)
          for s in tablewise_placement([rows[t] for t in tw_tabs], world)]
    placement = sorted(rw + tw, key=lambda s: (s.table_id, s.start))
    budget = 64 * D * 4
    model = (budget + 1000 + B, 1000, 1)
    cache = C.AdaptiveCache(budget, admission="sketch", record_evictions=True, max_dim=D, pooled_results=pooled)
    rk = ShardedRanker(metas, placement, 0, rank, world, f"cuda:{local}", tuple(range(len(rows))), ops, B,
                       params=RankerParams(pushdown_threshold=thr, admit_per_batch=8), cache=cache,
                       policy=C.CachePolicy(C.MemoryModel(*model)), tracker=C.LoadTracker(4, 10 ** 9, 0))
    pl = O.Placement.from_specs({m.table_id: m.num_rows for m in metas},
                                [(s.table_id, s.start, s.end, s.server_id) for s in placement])
    oc = O.CacheOracle(budget, admission="sketch", pooled=pooled)
    po = O.PipelineOracle(0, {m.table_id: D for m in metas}, pl, threshold=thr, cache=oc,
                          policy=O.CachePolicyO(O.MemoryModelO(*model)), tracker=O.LoadTrackerO(4, 10 ** 9, 0),
                          admit_per_batch=8)
    gen = DlrmBatchGen(rows, 1.1, B, (1, 6), seed=31 + rank, ops=ops)
    bad = {"metrics": 0, "counters": 0, "lru": 0, "tol": 0, "flat": 0}
    hits = raw = 0
    for it in range(8):
        hb = gen.next()
        pooled_out, cnt = rk.execute_csr(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(),
                                         batch_id=it)
        out = pooled_out.cpu().numpy()
        F = len(rows)
        bb = O.BagBatch(hb.offsets.astype(np.int64), hb.indices.astype(np.int64), np.repeat(np.arange(F), B),
                        [ops[f] for f in range(F) for _ in range(B)], np.tile(np.arange(B), F),
                        np.repeat(np.arange(F), B), B, it)
        vecs, counters, _ = po.run(bb)
        m, om = rk.batch_metrics[-1], po.metrics[-1]
        hits += m.cache_hits
        raw += m.raw_rows
        bad["metrics"] += (m.cache_hits, m.cache_misses, m.pushdown_groups, m.pushdown_rows, m.raw_rows) != \
            (om["hits"], om["misses"], om["pushdown_groups"], om["pushdown_rows"], om["raw_rows"])
        got_c = np.stack([cnt[k].cpu().numpy() for k in ("cache_hits", "pushdown_groups", "pushdown_rows",
                                                          "raw_rows")], 1)
        for b in range(F * B):
            f, s_ = divmod(b, B)
            bad["counters"] += tuple(int(x) for x in got_c[b]) != counters[b]
            g = out[s_, f * D:(f + 1) * D]
            bad["tol"] += not O.within_tolerance(vecs[b], g)
            flat = O.pool_flat(O.rows_of(0, f, D, hb.indices[hb.offsets[b]:hb.offsets[b + 1]]), ops[f])
            bad["flat"] += flat.tobytes() != g.tobytes()
        lru_gpu = [k if k[0] != "pooled" else ("pooled", k[1]) for k in rk.cache.lru_keys()]
        lru_ref = [k if k[0] != "pooled" else ("pooled", O.pooled_fingerprint(k[1], k[2], k[3])[0])
                   for k in oc.lru_keys()]
        bad["lru"] += lru_gpu != lru_ref
    ev_ok = [k for k in rk.cache.eviction_log if k[0] != "pooled"] == [k for k in oc.evictions if k[0] != "pooled"]
    t = torch.tensor([bad["metrics"], bad["counters"], bad["lru"], bad["tol"], bad["flat"], 0 if ev_ok else 1, hits, raw],
                     device="cpu" if fold else "cuda", dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"SHARDED_RANKER thr={thr} pooled={pooled} world={world} metric_mismatch_batches={t[0].item()} "
              f"counter_mismatches={t[1].item()} lru_mismatch_batches={t[2].item()} tolerance_failures={t[3].item()} "
              f"non_bit_exact_vs_flat={t[4].item()} eviction_log_mismatch={t[5].item()} "
              f"max_rank_cache_hits={t[6].item()} max_rank_raw_rows={t[7].item()}", flush=True)
    ok = int(t[:4].sum().item()) == 0 and t[5].item() == 0
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
