#!/bin/bash
# row-wise fused exchange with / without the reference plan (threshold 2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N=${N:-4}
for rep in 1; do
  for args in "--partial f64" "--partial f64 --threshold 2" "--partial f32" "--partial f32 --threshold 2" \
              "--partial f64 --sync" "--partial f64 --threshold 2 --sync"; do
    echo "== N=$N $args" >> gpurun_out/rwplan.log
    torchrun --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus $N --steps 100 \
      --warmup 10 --mode rowwise $args 2>>gpurun_out/rwplan.err | tail -1 >> gpurun_out/rwplan.log
  done
done
