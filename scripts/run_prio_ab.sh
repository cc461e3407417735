#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do for pr in 0 1; do
  FX_GATHER_PRIORITY=$pr torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2995$pr bench.py --gpus 4 --steps 300 \
    --warmup 10 --no-e2e 2>/dev/null | tail -1 > gpurun_out/prio_$pr.json
  echo "prio=$pr $(python -c "import json; d=json.load(open('gpurun_out/prio_$pr.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],4), d['roofline']['pool_ms_per_step_all_ranks'])")"
done; done
