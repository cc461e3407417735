#!/bin/bash
# D=64 K4 staging A/B on cfg1 (CUDA graph of 64 launches) and a large-batch D=64 cold control
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in 1 2; do
  FX_POOL_VARIANT=$v python bench.py --config cfg1 --graph 64 --steps 640 --warmup 64 --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/d64_$v.json
  echo "v=$v cfg1-graph $(python -c "import json; d=json.load(open('gpurun_out/d64_$v.json')); print(round(d['value']/1e6,1), round(d['roofline']['frac'],3))")"
done; done
