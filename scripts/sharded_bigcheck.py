"""Multi-GPU parity at the north star's sharded sizes (torchrun, one rank per GPU):

    torchrun --nproc-per-node N scripts/sharded_bigcheck.py cfg4r|cfg5|cfg5thr [--bags 2000] [--steps 3]

* cfg4r: 100 tables x 1M rows x 128, B=4096 per rank, L=20, Zipf 1.05,
  table-wise over the ranks, fused NVLink exchange, pipelined stream;
* cfg5: 200 tables x 1M rows x 128, B=4096 per rank, L=100, Zipf 1.0 with
  the fixed row permutation, row-wise over the ranks, f64 partials;
* cfg5thr: cfg5 with the reference's pushdown threshold 2 (singleton
  (bag, owner) groups raw-fetched over NVLink) and f32 partials.

Every rank pools its own batches; `--bags` sampled bags per rank and step
are checked bit-exact against the flat f64 pool of the CPU oracle (f64 and
table-wise modes) or within the reference tolerance (f32 partials), and for
cfg5thr the per-bag counters against the reference plan (pooling.py:88-100).
Prints one JSON line per rank-0 summary.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2410_12794_b200.sharded import P2PShardedLookup, rowwise_placement, tablewise_placement  # noqa: E402
from paper_2410_12794_b200.store import TableMeta  # noqa: E402
from paper_2410_12794_b200.workload import CONFIGS, DlrmBatchGen  # noqa: E402


def plan_counters(idx, placement_starts, placement_srv, threshold):
    """Reference plan per bag: groups per owner; >= threshold pushed down."""
    which = np.searchsorted(placement_starts, idx, side="right") - 1
    srv = placement_srv[which]
    pg = pr = raw = 0
    for s in np.unique(srv):
        n = int((srv == s).sum())
        if n >= threshold:
            pg += 1
            pr += n
        else:
            raw += n
    return pg, pr, raw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cfg4r", "cfg5", "cfg5thr"])
    ap.add_argument("--bags", type=int, default=2000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=None)
    a = ap.parse_args()
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
    cfg = dict(CONFIGS["cfg4r" if a.which == "cfg4r" else "cfg5"])
    rows, D = cfg["table_rows"], cfg["dim"]
    B = a.batch or cfg["batch"]
    F = len(rows)
    L = cfg["pooling"]
    metas = [TableMeta(t, n, D) for t, n in enumerate(rows)]
    mode = "tablewise" if a.which == "cfg4r" else "rowwise"
    placement = (tablewise_placement if mode == "tablewise" else rowwise_placement)(rows, world)
    thr = 2 if a.which == "cfg5thr" else None
    pdt = "f32" if a.which == "cfg5thr" else "f64"
    gens = DlrmBatchGen(rows, cfg["alpha"], B, (L, L) if isinstance(L, int) else L, seed=1000 * rank + 17,
                        permute=cfg.get("permute", False))
    hbs = [gens.next() for _ in range(a.steps)]
    max_nnz = int(max(int(h.offsets[-1]) for h in hbs) * 1.05) + 1024
    t0 = time.perf_counter()
    sl = P2PShardedLookup(metas, placement, 0, tuple(range(F)), ("sum",) * F, B, rank, world, f"cuda:{local}",
                          mode=mode, max_nnz=max_nnz, partial_dtype=pdt, pushdown_threshold=thr)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    dev_b = [(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda()) for h in hbs]
    outs, cnts = [], []
    for o in sl.stream(dev_b):
        outs.append(o.cpu().numpy().copy())
        if thr is not None:
            cnts.append(sl.counters().cpu().numpy().copy())
    sl._check()
    rng = np.random.default_rng(rank)
    starts = {t: np.array([s.start for s in sorted((s for s in placement if s.table_id == t), key=lambda s: s.start)])
              for t in range(F)}
    srvs = {t: np.array([s.server_id for s in sorted((s for s in placement if s.table_id == t),
                                                       key=lambda s: s.start)]) for t in range(F)}
    exact = checked = cnt_bad = 0
    worst = 0.0
    for it, hb in enumerate(hbs):
        for _ in range(a.bags):
            f, s_ = int(rng.integers(F)), int(rng.integers(B))
            b = f * B + s_
            ix = hb.indices[hb.offsets[b]:hb.offsets[b + 1]].astype(np.int64)
            ref = O.pool_flat(O.rows_of(0, f, D, ix), "sum")
            got = outs[it][s_, f * D:(f + 1) * D]
            exact += ref.tobytes() == got.tobytes()
            worst = max(worst, O.tolerance_ratio(ref, got))
            checked += 1
            if thr is not None:
                want = plan_counters(ix, starts[f], srvs[f], thr)
                cnt_bad += tuple(int(x) for x in cnts[it][:, b]) != want
    t = torch.tensor([worst, float(checked - exact), float(cnt_bad)], device="cpu" if fold else "cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"check": a.which, "world": world, "mode": mode, "partials": pdt, "threshold": thr,
                          "tables": F, "rows": rows[0], "batch_per_rank": B, "pooling": L,
                          "bags_checked_per_rank": checked, "max_non_bit_exact": int(t[1].item()),
                          "worst_tolerance_ratio": round(t[0].item(), 4), "counter_mismatches": int(t[2].item()),
                          "init_s": round(init_s, 1)}), flush=True)
    ok = t[0].item() <= 1.0 and t[2].item() == 0 and (pdt == "f32" or t[1].item() == 0)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
