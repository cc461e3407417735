"""Host<->device copy bandwidth on this box (pinned memory), for the e2e roofline."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
res = {}
if "--numa" in sys.argv:
    from paper_2410_12794_b200.numa import bind_to_device, device_local_cpus
    res["local_cpus"] = len(device_local_cpus(0))
    res["bound"] = len(bind_to_device(0))
res["cpus"] = len(os.sched_getaffinity(0))
for mb in (9.6, 54.5, 218):
    n = int(mb * 1e6 / 4)
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        res[f"{name}_{mb}MB_GBs"] = round(20 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)
# concurrent: H2D 9.6 MB and D2H 54.5 MB on two streams
h_in = torch.empty(int(9.6e6 / 4), dtype=torch.float32, pin_memory=True)
d_in = torch.empty_like(h_in, device=dev)
h_out = torch.empty(int(54.5e6 / 4), dtype=torch.float32, pin_memory=True)
d_out = torch.empty_like(h_out, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
torch.cuda.synchronize()
e1.record()
e1.synchronize()
res["concurrent_9.6in_54.5out_ms_per_pair"] = round(e0.elapsed_time(e1) / 20, 3)
print(json.dumps(res))
