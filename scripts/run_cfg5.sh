#!/bin/bash
cd "$(dirname "$0")/.."
for args in "--partial f64" "--partial f32" "--partial f32 --threshold 2"; do
  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29720 bench.py --gpus 4 --steps 30 --warmup 5 \
    --no-e2e --config cfg5 --mode rowwise $args 2>/dev/null | tail -1 > gpurun_out/cfg5.json
  echo "cfg5 N=4 $args $(python -c "import json; d=json.load(open('gpurun_out/cfg5.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), [round(x,2) for x in d['roofline']['pool_ms_per_step_all_ranks']], d['roofline']['frac'])")"
done
