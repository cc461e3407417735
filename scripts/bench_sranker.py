"""ShardedRanker throughput: cfg2 Criteo tables sharded over N GPUs, every
rank a ranker with its own GPU cache (threshold 2, sketch admission).

    torchrun --nproc-per-node N scripts/bench_sranker.py [--cache-pct 1] [--batches 8] [--warm 3]
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12794_b200 import cache as C  # noqa: E402
from paper_2410_12794_b200.ranker import RankerParams  # noqa: E402
from paper_2410_12794_b200.sharded import tablewise_placement  # noqa: E402
from paper_2410_12794_b200.sharded_ranker import ShardedRanker  # noqa: E402
from paper_2410_12794_b200.store import TableMeta  # noqa: E402
from paper_2410_12794_b200.workload import CRITEO_KAGGLE_ROWS, DlrmBatchGen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cache-pct", type=float, default=1.0)
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--threshold", default="2")
    ap.add_argument("--alpha", type=float, default=1.05)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    rows, D, B = CRITEO_KAGGLE_ROWS, 128, 4096
    F = len(rows)
    metas = [TableMeta(t, n, D) for t, n in enumerate(rows)]
    placement = tablewise_placement(rows, world)
    rows_cached = int(sum(rows) * a.cache_pct / 100)
    budget = rows_cached * D * 4
    cache = C.AdaptiveCache(budget, admission="sketch", max_dim=D, slot_capacity=rows_cached + 1,
                            sketch_capacity=4 * B * 40 * F)
    thr = None if a.threshold == "none" else int(a.threshold)
    rk = ShardedRanker(metas, placement, 0, rank, world, f"cuda:{local}", tuple(range(F)), ("sum",) * F, B,
                       params=RankerParams(pushdown_threshold=thr, admit_per_batch=64), cache=cache,
                       policy=C.CachePolicy(C.MemoryModel(budget + 1000 + B, 1000, 1)),
                       tracker=C.LoadTracker(16, 10 ** 9, 0), max_nnz=B * F * 41)
    gen = DlrmBatchGen(rows, a.alpha, B, (1, 40), seed=7 + rank)
    hbs = [gen.next() for _ in range(a.warm + a.batches)]
    dev_b = [(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda()) for h in hbs]
    times, hits = [], []
    rk.profile = True
    for i, (idx, offs) in enumerate(dev_b):
        if i == a.warm:
            rk.stage_ms = {}
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rk.execute_csr(idx, offs, batch_id=i)
        e1.record()
        e1.synchronize()
        if i >= a.warm:
            times.append(e0.elapsed_time(e1))
            hits.append(rk.batch_metrics[-1].hit_rate)
    t = torch.tensor([sum(times) / len(times)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        print(json.dumps({"what": "ShardedRanker (Ranker pipeline per GPU, own cache, sharded store)",
                          "n_gpus": world, "ms_per_batch_max_rank": round(ms, 3),
                          "pooled_lookups_per_s_total": world * B * F / (ms / 1e3),
                          "hit_rate_rank0": sum(hits) / len(hits), "cache_pct": a.cache_pct, "threshold": thr,
                          "alpha": a.alpha, "tables": "criteo-kaggle x128 table-wise", "per_gpu_batch": B,
                          "stage_ms_rank0": {k: round(v / len(times), 3) for k, v in rk.stage_ms.items()}}),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
