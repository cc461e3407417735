"""Fused batch step: parity against the vectorised oracle, and cfg3 timing.

    python scripts/step_check.py compare [--rows 1000000] [--batch 1024] [--alpha 0.6] [--cache 0.05] ...
    python scripts/step_check.py time [--rows 10000000] [--alpha 1.0] [--cache 0.02] [--batches 8] [--warm 3]

`compare` runs tests/step_harness.run_compare and prints one JSON line per
batch; `time` runs Ranker.execute_csr (sync=False, fused step + K4 on a side
stream) on the full cfg3 shape and reports ms per batch from CUDA events.
"""

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["compare", "time"])
    ap.add_argument("--tables", type=int, default=32)
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--pooling", type=int, default=20)
    ap.add_argument("--alpha", default="1.0")
    ap.add_argument("--cache", default=None, help="cache fraction(s) of all rows, comma-separated")
    ap.add_argument("--threshold", default="none")
    ap.add_argument("--admission", default="sketch")
    ap.add_argument("--batches", type=int, default=6)
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--sketch", type=int, default=8_000_000, help="AdaptiveCache sketch_capacity (table = 2x, pow2)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    thr = None if a.threshold == "none" else int(a.threshold)
    if a.mode == "compare":
        from step_harness import run_compare
        for alpha in [float(x) for x in a.alpha.split(",")]:
            for frac in [float(x) for x in (a.cache or "0.05").split(",")]:
                rep, _ = run_compare(tables=a.tables, rows=a.rows or 1_000_000, dim=a.dim, batch=a.batch or 1024,
                                     pooling=(a.pooling, a.pooling), alpha=alpha, cache_frac=frac, threshold=thr,
                                     admission=a.admission, n_batches=a.batches, depth=a.depth,
                                     fused=bool(a.fused), log=lambda r: print(json.dumps(r), flush=True))
                nbad = sum(len(r["bad"]) for r in rep)
                print(json.dumps({"alpha": alpha, "cache": frac, "threshold": thr, "batches": len(rep),
                                  "mismatches": nbad}), flush=True)
        return
    import paper_2410_12794_b200 as P
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams
    from paper_2410_12794_b200.workload import DlrmBatchGen
    T, N, D, B, L = a.tables, a.rows or 10_000_000, a.dim, a.batch or 4096, a.pooling
    metas = [P.TableMeta(t, N, D) for t in range(T)]
    placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
    dep = P.init_store(metas, placement, 0)
    for alpha in [float(x) for x in a.alpha.split(",")]:
        gen = DlrmBatchGen((N,) * T, alpha, B, (L, L), seed=7)
        hbs = [gen.next() for _ in range(a.warm + a.batches)]
        dbs = [(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda()) for h in hbs]
        for frac in [float(x) for x in (a.cache or "0.01,0.02").split(",")]:
            rows_c = int(T * N * frac)
            budget = rows_c * D * 4
            cache = C.AdaptiveCache(budget, admission=a.admission, max_dim=D, slot_capacity=rows_c + 1,
                                    sketch_capacity=a.sketch)
            rk = Ranker(dep, P.build_routing(metas, placement), None,
                        RankerParams(pushdown_threshold=thr, admit_per_batch=64, pipeline_depth=a.depth),
                        cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1_000 + B, 1_000, 1)),
                        tracker=C.LoadTracker(16, 10 ** 9, 0), fused=bool(a.fused))
            times = []
            rk.profile = True
            for i, (idx, offs) in enumerate(dbs):
                if i == a.warm:
                    rk.stage_ms = {}
                h = hbs[i]
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                rk.execute_csr(idx, offs, h.feature_tables, h.feature_ops, B, batch_id=i, sync=False)
                e1.record()
                e1.synchronize()
                if i >= a.warm:
                    times.append(e0.elapsed_time(e1))
            rk.sync()
            hr = [m.hit_rate for m in rk.batch_metrics[a.warm:]]
            sc = rk._step.scalars(0) if rk._step is not None else {}
            ms = sum(times) / len(times)
            print(json.dumps({"alpha": alpha, "cache_frac": frac, "cache_rows": rows_c, "ms_per_batch": round(ms, 4),
                              "bags_per_s": B * T / (ms / 1e3), "hit_rate": sum(hr) / len(hr),
                              "latency_ms": [round(m.latency * 1e3, 3) for m in rk.batch_metrics[a.warm:]],
                              "last_step": {k: sc.get(k) for k in ("n_uniq", "n_cand", "n_off", "n_hard", "n_rej",
                                                                   "n_acc", "n_ev", "mode", "F", "n_levels",
                                                                   "chain_cycles", "stage_on", "topk_fast", "topk_live", "topk_n")},
                              "capacity": cache.capacity(),
                              "phase_ms_per_batch": {k: round(v / max(1, len(times)), 3)
                                                     for k, v in rk.stage_ms.items()},
                              "fused": bool(a.fused), "threshold": thr}), flush=True)
            del rk, cache
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
