"""Many small concurrent requests on one GPU (SURVEY §8(d) cfg5's "64
concurrent request streams x 64 samples", §8(f) rank 1): per-request K4
launches vs LookupEngine.pool_many (one launch for all requests) vs a CUDA
graph of the per-request launches, on the cfg2 tables.

    python scripts/bench_multireq.py [--requests 64] [--samples 64] [--iters 50]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_12794_b200 as P  # noqa: E402
from paper_2410_12794_b200.workload import CRITEO_KAGGLE_ROWS, DlrmBatchGen  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--samples", type=int, default=64)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rows, D = CRITEO_KAGGLE_ROWS, 128
    F = len(rows)
    dep = P.init_store([P.TableMeta(t, n, D) for t, n in enumerate(rows)],
                       [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(rows)], seed=0)
    eng = P.LookupEngine(dep)
    reqs = []
    for r in range(a.requests):
        hb = DlrmBatchGen(rows, 1.05, a.samples, (1, 40), seed=1000 + r).next()
        reqs.append(P.CsrBatch(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda(),
                               hb.feature_tables, hb.feature_ops, hb.batch_size))
    outs = [torch.empty((a.samples, F * D), dtype=torch.float32, device="cuda") for _ in reqs]
    bags = a.requests * a.samples * F

    def per_request():
        for b, o in zip(reqs, outs):
            eng.pool(b, out=o, check=False)

    plan = eng.prepare_many(reqs, outs)

    def many():
        plan.launch()

    g = eng.capture(reqs, outs)
    res = {"requests": a.requests, "samples_per_request": a.samples, "tables": "criteo-kaggle 26 x 128",
           "bags_per_round": bags}
    for name, fn in (("per_request_launches", per_request), ("pool_many_one_launch", many),
                     ("cuda_graph_of_launches", g.replay)):
        ms = timed(fn, a.iters)
        res[name] = {"ms": round(ms, 4), "bags_per_s": bags / (ms / 1e3)}
    big = DlrmBatchGen(rows, 1.05, a.requests * a.samples, (1, 40), seed=7).next()
    bb = P.CsrBatch(torch.from_numpy(big.indices).cuda(), torch.from_numpy(big.offsets).cuda(), big.feature_tables,
                    big.feature_ops, big.batch_size)
    ob = torch.empty((big.batch_size, F * D), dtype=torch.float32, device="cuda")
    ms = timed(lambda: eng.pool(bb, out=ob, check=False), a.iters)
    res["one_batch_same_samples"] = {"ms": round(ms, 4), "bags_per_s": bags / (ms / 1e3)}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
