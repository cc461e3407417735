#!/bin/bash
# cfg5 row-wise at N=4: per-rank pool imbalance diagnosis (priority stream,
# pipelining, partial dtype)
O=gpurun_out/m4diag
mkdir -p $O
N=$(python -c "import torch; print(torch.cuda.device_count())")
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --config cfg5 --mode rowwise --no-cpu --no-e2e > $O/base.json 2> $O/base.err
FX_GATHER_PRIORITY=0 timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --config cfg5 --mode rowwise --no-cpu --no-e2e > $O/noprio.json 2> $O/noprio.err
timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --config cfg5 --mode rowwise --no-cpu --no-e2e --sync > $O/sync.json 2> $O/sync.err
timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --config cfg5 --mode rowwise --no-cpu --no-e2e --partial f32 > $O/f32.json 2> $O/f32.err
echo done
