"""e2e host-API variants at cfg2 (pinned CSR in, pinned pooled out)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_12794_b200 as P  # noqa: E402
from paper_2410_12794_b200.engine import CsrBatch, HostLookup, LookupEngine  # noqa: E402
from bench import build_cfg  # noqa: E402

torch.cuda.set_device(0)
cfg, host_batches = build_cfg("cfg2", 0, 4, None, None)
dim = cfg["dim"]
metas = [P.TableMeta(t, n, dim) for t, n in enumerate(cfg["table_rows"])]
dep = P.init_store(metas, [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(cfg["table_rows"])], seed=0)
eng = LookupEngine(dep)
hl = HostLookup(eng)
pinned = [CsrBatch(torch.from_numpy(hb.indices).pin_memory(), torch.from_numpy(hb.offsets).pin_memory(),
                   hb.feature_tables, hb.feature_ops, hb.batch_size) for hb in host_batches]
bags = cfg["batch"] * len(cfg["table_rows"])
res = {}
for depth in (2, 3, 4, 6):
    for _ in hl.stream([pinned[i % 4] for i in range(6)], depth=depth):
        pass
    torch.cuda.synchronize()
    K = 60
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in hl.stream([pinned[i % 4] for i in range(K)], depth=depth):
        pass
    e1.record()
    e1.synchronize()
    res[f"depth{depth}_Mbags"] = round(bags * K / (e0.elapsed_time(e1) / 1e3) / 1e6, 1)
print(json.dumps(res), flush=True)
