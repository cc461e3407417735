#!/bin/bash
# default bench at N=2 and N=4 (value + e2e through stream_host)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in 2 4; do
  torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2968$n bench.py --gpus $n --steps 200 \
    --warmup 10 2>>gpurun_out/e2e_scale.err | tail -1 > gpurun_out/e2e_n$n.json
done
