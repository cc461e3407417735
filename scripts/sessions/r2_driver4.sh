#!/bin/bash
# the driver's N=4 invocations, as it launches them: our arm (defaults) and the reference arm
O=gpurun_out/d4
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641"
timeout 900 $R bench.py --impl reference --gpus 4 --steps 5 --warmup 3 > $O/ref.json 2> $O/ref.err; echo "rc=$?" >> $O/ref.err
timeout 900 $R bench.py --gpus 4 --steps 50 --warmup 5 > $O/ours.json 2> $O/ours.err; echo "rc=$?" >> $O/ours.err
echo done
