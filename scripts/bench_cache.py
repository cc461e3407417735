"""cfg3-shaped hot-cache sweep on one B200 (SURVEY §8(d) cfg3 semantics).

    python scripts/bench_cache.py [--tables 32] [--rows 10000000] [--alphas 0.6,0.8,1.0,1.2]
                                  [--cache-pct 1,2,5] [--batches 6] [--warm 3]

Ranker with the GPU cache, pushdown threshold None (every miss raw-fetched
and offered), sketch admission, admit_per_batch 64, adaptive maintenance
with the memory model pinned so the budget stays at the swept size. Prints
one JSON line per (alpha, cache%): steady-state hit rate, per-batch device
time of the whole pipeline, and pooled lookups/s.
"""

import argparse
import gc
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_12794_b200 as P  # noqa: E402
from paper_2410_12794_b200 import cache as C  # noqa: E402
from paper_2410_12794_b200.ranker import Ranker, RankerParams  # noqa: E402
from paper_2410_12794_b200.workload import DlrmBatchGen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tables", type=int, default=32)
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--pooling", default="20", help="L, or lo,hi for ragged bags")
    ap.add_argument("--pooled", type=int, default=0, help="pooled-result keyspace on (cache.py:204-223)")
    ap.add_argument("--threshold", default="none", help="pushdown threshold (none or an int >= 2)")
    ap.add_argument("--alphas", default="0.6,0.8,1.0,1.2")
    ap.add_argument("--cache-pct", default="1,2,5")
    ap.add_argument("--batches", type=int, default=6)
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--hits-from-cache", type=int, default=0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    T, N, D, B = a.tables, a.rows, a.dim, a.batch
    pool = tuple(int(x) for x in a.pooling.split(","))
    pool = pool if len(pool) == 2 else (pool[0], pool[0])
    thr = None if a.threshold == "none" else int(a.threshold)
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    t0 = time.perf_counter()
    dep = P.init_store(metas, placement, 0)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    for alpha in [float(x) for x in a.alphas.split(",")]:
        gen = DlrmBatchGen((N,) * T, alpha, B, pool, seed=7)
        batches = [gen.next() for _ in range(a.warm + a.batches)]
        dev_batches = [(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda())
                       for hb in batches]
        for pct in [float(x) for x in a.cache_pct.split(",")]:
            rows_cached = int(T * N * pct / 100)
            free, total = torch.cuda.mem_get_info()
            print(f"alpha {alpha} cache {pct}%: {free / 2**30:.1f} of {total / 2**30:.1f} GiB free", file=sys.stderr)
            budget = rows_cached * D * 4
            per_sample = 1
            model = C.MemoryModel(budget + 1_000 + B * per_sample, 1_000, per_sample)
            cache = C.AdaptiveCache(budget, admission="sketch", max_dim=D, slot_capacity=rows_cached + 1,
                                    sketch_capacity=4 * B * pool[1] * T, pooled_results=bool(a.pooled))
            rk = Ranker(dep, P.build_routing(metas, placement), None,
                        RankerParams(pushdown_threshold=thr, admit_per_batch=64), cache=cache,
                        policy=C.CachePolicy(model), tracker=C.LoadTracker(16, 10 ** 9, 0),
                        hits_from_cache=bool(a.hits_from_cache))
            times, hits = [], []
            rk.profile = True
            for i, (idx, offs) in enumerate(dev_batches):
                torch.cuda.synchronize()
                if i == a.warm:
                    rk.stage_ms = {}
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rk.execute_csr(idx, offs, batches[i].feature_tables, batches[i].feature_ops, B, batch_id=i)
                e1.record()
                e1.synchronize()
                if i >= a.warm:
                    times.append(e0.elapsed_time(e1))
                    hits.append(rk.batch_metrics[-1].hit_rate)
            ms = sum(times) / len(times)
            print(json.dumps({"alpha": alpha, "cache_pct": pct, "cache_rows": rows_cached,
                              "hit_rate": sum(hits) / len(hits), "ms_per_batch": ms,
                              "pooled_lookups_per_s": B * T / (ms / 1e3), "tables": T, "rows": N, "dim": D,
                              "batch": B, "pooling": list(pool), "init_store_s": round(init_s, 2),
                              "pooled_keyspace": bool(a.pooled), "threshold": thr,
                              "pooled_hit_bags_last": getattr(rk, "last_pooled_hits", None),
                              "offer_tiles": {k: cache._scalars()[k] for k in ("tiles_bulk", "tiles_chain")},
                              "hits_from_cache": bool(a.hits_from_cache),
                              "stage_ms_per_batch": {k: round(v / len(times), 3) for k, v in rk.stage_ms.items()}}),
                  flush=True)
            del rk, cache
            gc.collect()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
