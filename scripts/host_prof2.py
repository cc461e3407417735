"""Host time of each piece of Ranker.execute_csr(sync=False) (cfg3 shape)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_12794_b200 as P  # noqa: E402
from paper_2410_12794_b200 import cache as C  # noqa: E402
from paper_2410_12794_b200 import step as S  # noqa: E402
from paper_2410_12794_b200.ranker import Ranker, RankerParams  # noqa: E402
from paper_2410_12794_b200.workload import DlrmBatchGen  # noqa: E402

T, N, D, B, L = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000, 128, 4096, 20
metas = [P.TableMeta(t, N, D) for t in range(T)]
placement = [P.ShardSpec(t, 0, N, 0) for t in range(T)]
dep = P.init_store(metas, placement, 0)
gen = DlrmBatchGen((N,) * T, 1.0, B, (L, L), seed=7)
hbs = [gen.next() for _ in range(16)]
dbs = [(torch.from_numpy(h.indices).cuda(), torch.from_numpy(h.offsets).cuda()) for h in hbs]
rows_c = int(T * N * 0.02)
budget = rows_c * D * 4
cache = C.AdaptiveCache(budget, max_dim=D, slot_capacity=rows_c + 1, sketch_capacity=8_000_000)
rk = Ranker(dep, P.build_routing(metas, placement), None, RankerParams(pushdown_threshold=None),
            cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1_000 + B, 1_000, 1)),
            tracker=C.LoadTracker(16, 10 ** 9, 0))
acc = {}


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return r
    setattr(obj, name, g)


for i in range(6):
    rk.execute_csr(*dbs[i], hbs[i].feature_tables, hbs[i].feature_ops, B, batch_id=i, sync=False)
rk.sync()
torch.cuda.synchronize()
for n in ("start", "offer", "maintain", "scalars_tensor"):
    wrap(rk._step, n)
for n in ("_pool_sample_major", "_fast_start", "_fast_finish", "_get_step"):
    wrap(rk, n)
t0 = time.perf_counter()
for i in range(6, 16):
    rk.execute_csr(*dbs[i], hbs[i].feature_tables, hbs[i].feature_ops, B, batch_id=i, sync=False)
host = (time.perf_counter() - t0) / 10
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 10
print("host ms/batch", round(host * 1e3, 3), "wall ms/batch", round(wall * 1e3, 3))
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:22s} {v / 10 * 1e3:8.3f} ms")
