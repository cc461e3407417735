"""torchrun --nproc-per-node N scripts/sharded_check.py [tablewise|rowwise] [exchange]
Sharded lookup on N GPUs vs the CPU oracle (flat f64 pool) for every rank's batch.

FX_FOLD_DEVICES=1 folds the ranks onto the visible GPUs (rank r on device
r % count; a one-GPU box runs every rank on cuda:0): the fused exchange then
goes through same-device CUDA-IPC mappings of the other ranks' buffers, the
control plane uses gloo, and the NCCL exchange is not available."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2410_12794_b200.sharded import (P2PShardedLookup, ShardedLookup, rowwise_placement,  # noqa: E402
                                           tablewise_placement)
from paper_2410_12794_b200.store import TableMeta  # noqa: E402
from paper_2410_12794_b200.workload import DlrmBatchGen  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "tablewise"
    exchange = sys.argv[2] if len(sys.argv) > 2 else "nccl"
    hosted = exchange.endswith("-host")  # pinned host in/out through stream_host
    pipelined = exchange.endswith("-pipe") or hosted
    exchange = exchange[:-5] if pipelined else exchange
    fold = os.environ.get("FX_FOLD_DEVICES") == "1"
    local = int(os.environ["LOCAL_RANK"]) % (torch.cuda.device_count() if fold else 1 << 30)
    torch.cuda.set_device(local)
    if fold:
        if exchange == "nccl":
            raise SystemExit("the NCCL exchange needs one GPU per rank (FX_FOLD_DEVICES folds ranks onto one GPU)")
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    rows = (50_000, 123, 20_000, 7, 9_999, 100_000, 31, 4_096, 64, 2)
    ops = ("sum", "mean") * 5
    D, B = 128, 96
    metas = [TableMeta(t, n, D) for t, n in enumerate(rows)]
    placement = (tablewise_placement if mode == "tablewise" else rowwise_placement)(rows, world)
    if exchange == "p2phybrid":
        from paper_2410_12794_b200.store import ShardSpec
        repl = [t for t, n in enumerate(rows) if n < 5000]
        big = [t for t in range(len(rows)) if t not in repl]
        sub = tablewise_placement([rows[t] for t in big], world)
        placement = [ShardSpec(big[s.table_id], s.start, s.end, s.server_id) for s in sub]
        sl = P2PShardedLookup(metas, placement, 0, tuple(range(len(rows))), ops, B, rank, world, f"cuda:{local}",
                              mode=mode, replicated_tables=repl)
    elif exchange in ("p2pthr", "p2pthr32"):
        # reference plan: groups < 2 raw-fetched over NVLink, larger ones pushed down
        sl = P2PShardedLookup(metas, placement, 0, tuple(range(len(rows))), ops, B, rank, world, f"cuda:{local}",
                              mode=mode, partial_dtype="f32" if exchange == "p2pthr32" else "f64",
                              pushdown_threshold=2)
    elif exchange == "p2pf32":
        sl = P2PShardedLookup(metas, placement, 0, tuple(range(len(rows))), ops, B, rank, world, f"cuda:{local}",
                              mode=mode, partial_dtype="f32")
    elif exchange == "p2p":
        # per-rank staging requirement differs (ragged batches): the class must agree on one geometry
        sl = P2PShardedLookup(metas, placement, 0, tuple(range(len(rows))), ops, B, rank, world, f"cuda:{local}",
                              mode=mode, max_nnz=B * len(rows) * 40 + 97 * rank)
    else:
        sl = ShardedLookup(metas, placement, 0, tuple(range(len(rows))), ops, B, rank, world, f"cuda:{local}",
                           mode=mode)
    worst, exact, n = 0.0, 0, 0
    hbs = [DlrmBatchGen(rows, 1.0, B, (1, 40), seed=100 * rank + it, ops=ops, permute=(mode == "rowwise")).next()
           for it in range(4)]
    if pipelined:
        dev_b = [(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda()) for hb in hbs]
        torch.cuda.synchronize()
        outs, cnts = [], []
        if hosted:
            dev_b = [(torch.from_numpy(hb.indices).pin_memory(), torch.from_numpy(hb.offsets).pin_memory())
                     for hb in hbs]
        for o in (sl.stream_host(dev_b) if hosted else sl.stream(dev_b)):
            outs.append(o.cpu().numpy().copy())
            if exchange.startswith("p2pthr"):
                cnts.append(sl.counters().cpu().numpy())
    planned = exchange.startswith("p2pthr")
    hier_exact = cnt_bad = 0
    if planned:
        pl = O.Placement.from_specs({m.table_id: m.num_rows for m in metas},
                                    [(sp.table_id, sp.start, sp.end, sp.server_id) for sp in placement])
        po = O.PipelineOracle(0, {m.table_id: D for m in metas}, pl, threshold=2)
    for it in range(4):
        hb = hbs[it]
        if pipelined:
            out = outs[it]
        else:
            out = sl.lookup(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda()).cpu().numpy()
        if planned:
            cnt = cnts[it] if pipelined else sl.counters().cpu().numpy()
            nb = len(rows) * B
            bb = O.BagBatch(hb.offsets.astype(np.int64), hb.indices.astype(np.int64),
                            np.repeat(np.arange(len(rows)), B), [ops[f] for f in range(len(rows)) for _ in range(B)],
                            np.tile(np.arange(B), len(rows)), np.repeat(np.arange(len(rows)), B), B)
            vecs, counters, _ = po.run(bb)
            for b in range(nb):
                f, s_ = divmod(b, B)
                cnt_bad += tuple(int(x) for x in cnt[:, b]) != counters[b][1:]
                if exchange == "p2pthr32":  # f32 partials + raw rows: the reference's own combine
                    hier_exact += vecs[b].tobytes() != out[s_, f * D:(f + 1) * D].tobytes()
        for f in range(len(rows)):
            for s in range(B):
                b = f * B + s
                ref = O.pool_flat(O.rows_of(0, f, D, hb.indices[hb.offsets[b]:hb.offsets[b + 1]]), ops[f])
                got = out[s, f * D:(f + 1) * D]
                worst = max(worst, O.tolerance_ratio(ref, got))
                exact += ref.tobytes() == got.tobytes()
                n += 1
    # edge cases: a batch whose bags are all empty, and one with every other bag empty
    empty_bad = 0.0
    if not pipelined and exchange in ("p2p", "nccl", "p2pf32", "p2phybrid"):
        F = len(rows)
        offs0 = torch.zeros(F * B + 1, dtype=torch.int64, device="cuda")
        o = sl.lookup(torch.zeros(0, dtype=torch.int32, device="cuda"), offs0).cpu().numpy()
        empty_bad += float(np.abs(o).max()) if o.size else 0.0
        hb = hbs[1]
        lens = np.diff(hb.offsets)
        keep = np.arange(F * B) % 2 == 0
        new_lens = np.where(keep, lens, 0)
        new_offs = np.concatenate([[0], np.cumsum(new_lens)]).astype(np.int64)
        new_idx = np.concatenate([hb.indices[hb.offsets[b]:hb.offsets[b + 1]] for b in range(F * B) if keep[b]])
        o = sl.lookup(torch.from_numpy(new_idx).cuda(), torch.from_numpy(new_offs).cuda()).cpu().numpy()
        for b in range(F * B):
            f, s_ = divmod(b, B)
            got = o[s_, f * D:(f + 1) * D]
            if keep[b]:
                ref = O.pool_flat(O.rows_of(0, f, D, new_idx[new_offs[b]:new_offs[b + 1]]), ops[f])
                empty_bad += 0.0 if O.within_tolerance(ref, got) else 1.0
            else:
                empty_bad += float(np.abs(got).max())
    # ingress validation (ranker.py:184-193): an out-of-range index on rank 1's
    # batch raises LookupValidationError there; every rank recovers next step
    val_bad = 0.0
    if exchange in ("p2p", "nccl") and not pipelined and world > 1:
        from paper_2410_12794_b200.errors import LookupValidationError, RoutingViolationError
        hb = hbs[0]
        idx = hb.indices.copy()
        if rank == 1:
            idx[hb.offsets[3 * B + 5]] = rows[3] + 7  # table 3, sample 5
        got = None
        try:
            sl.lookup(torch.from_numpy(idx).cuda(), torch.from_numpy(hb.offsets).cuda())
        except (LookupValidationError, RoutingViolationError) as e:
            got = type(e).__name__
        if rank == 1 and got != "LookupValidationError":
            val_bad = 1.0
        dist.barrier()
        out = sl.lookup(torch.from_numpy(hb.indices).cuda(), torch.from_numpy(hb.offsets).cuda()).cpu().numpy()
        ref = O.pool_flat(O.rows_of(0, 0, D, hb.indices[hb.offsets[0]:hb.offsets[1]]), ops[0])
        val_bad += 0.0 if O.within_tolerance(ref, out[0, :D]) else 1.0
    t = torch.tensor([worst, float(n - exact), float(cnt_bad), float(hier_exact), val_bad, empty_bad],
                     device="cpu" if fold else "cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"SHARDED {mode} {exchange}{('-host' if hosted else '-pipe') if pipelined else ''} world={world} worst_tolerance_ratio={t[0].item():.4f} "
              f"max_non_bit_exact_bags={int(t[1].item())} bags_per_rank={n} counter_mismatches={int(t[2].item())} "
              f"non_bit_exact_vs_reference_combine={int(t[3].item())} validation_failures={int(t[4].item())} "
              f"empty_bag_failures={t[5].item():g}", flush=True)
    ok = t[0].item() <= 1.0 and t[2].item() == 0 and t[3].item() == 0 and t[4].item() == 0 and t[5].item() == 0
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
