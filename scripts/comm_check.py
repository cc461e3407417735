"""fx_alltoallv (PeerComm, CUDA-IPC peer stores) vs NCCL all_to_all_single on
random ragged byte counts, several consecutive exchanges (the double-buffered
windows), plus bandwidth at a pooled-return-sized exchange.

    torchrun --nproc-per-node N scripts/comm_check.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2410_12794_b200.sharded import PeerComm
    rank, world = dist.get_rank(), dist.get_world_size()
    slot = 1 << 20
    comm = PeerComm(slot)
    g = torch.Generator().manual_seed(1234 + rank)
    for it in range(6):
        # every count a multiple of 4 except some ragged tails (byte path)
        counts = torch.randint(0, slot + 1, (world,), generator=g)
        if it % 2:
            counts[0] = counts[0] - counts[0] % 16 + 7  # unaligned tail
        counts = counts.clamp(0, slot)
        displs = torch.zeros(world, dtype=torch.int64)
        displs[1:] = torch.cumsum(counts, 0)[:-1]
        send = torch.randint(0, 256, (int(counts.sum()),), dtype=torch.uint8, generator=g).cuda()
        recv, rcounts = comm.alltoallv(send, counts.cuda(), displs.cuda())
        # NCCL reference: exchange counts, then the bytes
        in_counts = torch.empty(world, dtype=torch.int64, device="cuda")
        dist.all_to_all_single(in_counts, counts.cuda())
        ref = torch.empty(int(in_counts.sum()), dtype=torch.uint8, device="cuda")
        dist.all_to_all_single(ref, send, in_counts.tolist(), counts.tolist())
        torch.cuda.synchronize()
        assert torch.equal(rcounts.cpu(), in_counts.cpu()), (rcounts, in_counts)
        off = 0
        for s in range(world):
            n = int(in_counts[s])
            assert torch.equal(recv[s, :n], ref[off:off + n]), (it, s)
            off += n
    ov, to = comm.status()
    assert ov == 0 and to == 0
    # bandwidth: every rank sends slot bytes to every other rank
    big = 64 << 20
    comm2 = PeerComm(big)
    counts = torch.full((world,), big, dtype=torch.int64, device="cuda")
    displs = torch.arange(world, dtype=torch.int64, device="cuda") * big
    send = torch.ones(world * big, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        comm2.alltoallv(send, counts, displs)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        comm2.alltoallv(send, counts, displs)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # per rank: (world - 1) * big bytes over NVLink out (+ the same in), plus the local slot
    gbs = (world - 1) * big / (ms.item() / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({"check": "fx_alltoallv", "world": world, "exchanges_checked": 6,
                          "bw_bytes_per_peer": big, "ms": round(ms.item(), 4),
                          "nvlink_out_gbs_per_gpu": round(gbs, 1)}), flush=True)
        print(f"COMM OK world={world}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
