"""Host-side profile of Ranker.execute_csr(sync=False) on a cfg3 shape (cProfile)."""
import cProfile
import os
import pstats
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_12794_b200 as P  # noqa: E402
from paper_2410_12794_b200 import cache as C  # noqa: E402
from paper_2410_12794_b200.ranker import Ranker, RankerParams  # noqa: E402
from paper_2410_12794_b200.workload import DlrmBatchGen  # noqa: E402

T, N, D, B, L = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000, 128, 4096, 20
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
metas = [P.TableMeta(t, N, D) for t in range(T)]
placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
dep = P.init_store(metas, placement, 0)
gen = DlrmBatchGen((N,) * T, alpha, B, (L, L), seed=7)
hbs = [gen.next() for _ in range(12)]
dbs = [(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda()) for h in hbs]
rows_c = int(T * N * 0.02)
budget = rows_c * D * 4
cache = C.AdaptiveCache(budget, max_dim=D, slot_capacity=rows_c + 1, sketch_capacity=8_000_000)
rk = Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=None),
            cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1_000 + B, 1_000, 1)),
            tracker=C.LoadTracker(16, 10 ** 9, 0))
for i in range(3):
    rk.execute_csr(*dbs[i], hbs[i].feature_tables, hbs[i].feature_ops, B, batch_id=i, sync=False)
rk.sync()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for i in range(3, 12):
    t1 = time.perf_counter()
    rk.execute_csr(*dbs[i], hbs[i].feature_tables, hbs[i].feature_ops, B, batch_id=i, sync=False)
    print("host ms", round((time.perf_counter() - t1) * 1e3, 3), flush=True)
pr.disable()
torch.cuda.synchronize()
print("wall per batch ms", (time.perf_counter() - t0) / 9 * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
