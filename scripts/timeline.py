"""Real-time kernel timeline of captured Ranker batches (cfg3 bench setup):
torch.profiler (CUPTI activity records, not serialised like ncu) over a few
graph replays; prints per-step span, busy time on each stream, idle gaps and
the top kernels by wall time, as one JSON line.

    python scripts/timeline.py [--alpha 1.0] [--cache 0.02] [--warm 12] [--steps 4]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--cache", type=float, default=0.02)
    ap.add_argument("--warm", type=int, default=12)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--rows", type=int, default=10_000_000)
    a = ap.parse_args()
    import paper_2410_12794_b200 as P
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen
    T, N, D, B, L = 32, a.rows, 128, 4096, 20
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    dep = P.init_store(metas, placement, 0)
    gen = DlrmBatchGen((N,) * T, a.alpha, B, (L, L), seed=7)
    hbs = [gen.next() for _ in range(a.warm + a.steps + 2)]
    dbs = [(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda()) for h in hbs]
    ft, fo = hbs[0].feature_tables, hbs[0].feature_ops
    rows_c = int(T * N * a.cache)
    budget = rows_c * D * 4
    cache = C.AdaptiveCache(budget, admission="sketch", max_dim=D, slot_capacity=rows_c + 1,
                            sketch_capacity=8_000_000)
    rk = Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=None, admit_per_batch=64),
                cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1_000 + B, 1_000, 1)),
                tracker=C.LoadTracker(16, 10 ** 9, 0))
    for i in range(a.warm):
        rk.execute_csr(*dbs[i], ft, fo, B, batch_id=i, sync=False)
    rk.sync()
    sidx, soffs = dbs[0][0].clone(), dbs[0][1].clone()
    g = rk.capture_csr(sidx, soffs, ft, fo, B)
    for i in range(2):
        sidx.copy_(dbs[a.warm + i][0])
        soffs.copy_(dbs[a.warm + i][1])
        g.replay(batch_id=-1 - i)
    rk.sync()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(a.steps):
            j = a.warm + 2 + i if a.warm + 2 + i < len(dbs) else a.warm
            sidx.copy_(dbs[j][0])
            soffs.copy_(dbs[j][1])
            g.replay(batch_id=100 + i)
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        evs.append((e.time_range.start, e.time_range.end, e.name, getattr(e, "device_resource_id", 0)))
    evs.sort()
    # steps: split at the D2D copy into sidx (a Memcpy DtoD before each replay)
    starts = [s for s, _, n, _ in evs if "ks_begin" in n]
    spans = []
    per_kernel = {}
    for k in range(len(starts)):
        lo = starts[k]
        hi = starts[k + 1] if k + 1 < len(starts) else max(e for _, e, _, _ in evs)
        seg = [x for x in evs if lo <= x[0] < hi]
        end = max(e for _, e, _, _ in seg)
        # union of busy intervals
        busy, cur_s, cur_e = 0.0, None, None
        for s, e, _, _ in sorted(seg):
            if cur_e is None or s > cur_e:
                if cur_e is not None:
                    busy += cur_e - cur_s
                cur_s, cur_e = s, e
            else:
                cur_e = max(cur_e, e)
        busy += cur_e - cur_s
        spans.append({"span_us": round(end - lo, 1), "busy_us": round(busy, 1), "kernels": len(seg)})
        if k > 0:
            for s, e, n, _ in seg:
                nm = n.split("(")[0].replace("void ", "")
                nm = nm.split("<")[0] if nm.startswith("fx::") else nm[:60]
                per_kernel[nm] = per_kernel.get(nm, 0.0) + (e - s) / max(1, len(starts) - 1)
    top = sorted(per_kernel.items(), key=lambda kv: -kv[1])[:30]
    if len(starts) > 2:  # one step's timeline: (start offset us, duration us, stream, kernel)
        lo, hi = starts[1], starts[2]
        for s, e, n, r in [x for x in evs if lo <= x[0] < hi]:
            print(f"{s - lo:8.1f} {e - s:7.1f} {r:>4} {n[:90]}", file=sys.stderr)
    print(json.dumps({"alpha": a.alpha, "cache": a.cache, "steps": spans,
                      "kernel_sum_us": round(sum(per_kernel.values()), 1),
                      "top": [(k, round(v, 1)) for k, v in top]}), flush=True)


if __name__ == "__main__":
    main()
