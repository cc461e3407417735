"""One-GPU run of the row-wise fused exchange on a cfg5-shaped batch (for an
ncu launch list of the stage / gather / combine kernels)."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12794_b200.sharded import P2PShardedLookup, rowwise_placement  # noqa: E402
from paper_2410_12794_b200.store import TableMeta  # noqa: E402
from paper_2410_12794_b200.workload import DlrmBatchGen  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29931")
dist.init_process_group("gloo", rank=0, world_size=1)
torch.cuda.set_device(0)
T = int(os.environ.get("TABLES", "50"))
rows = (1_000_000,) * T
B, D = 4096, 128
metas = [TableMeta(t, n, D) for t, n in enumerate(rows)]
sl = P2PShardedLookup(metas, rowwise_placement(rows, 1), 0, tuple(range(T)), ("sum",) * T, B, 0, 1, "cuda:0",
                      mode="rowwise", partial_dtype="f32", max_nnz=B * T * 100 + 1024)
hb = DlrmBatchGen(rows, 1.0, B, 100, seed=1, permute=True).next()
idx, offs = torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda()
for _ in range(3):
    sl.lookup(idx, offs)
torch.cuda.synchronize()
print("ok", hb.indices.size)
