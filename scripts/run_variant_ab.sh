#!/bin/bash
# K4 variant A/B on cfg2 and the cold control
cd "$(dirname "$0")/.."
VARS=${VARS:-"1 2"}
for v in $VARS; do FX_POOL_VARIANT=$v python -m pytest tests/test_gpu_core.py -q -x 2>&1 | tail -1; done
for rep in 1 2; do
for v in $VARS; do
  FX_POOL_VARIANT=$v python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/ab_cfg2_$v.json
  FX_POOL_VARIANT=$v python bench.py --steps 100 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 2>/dev/null | tail -1 > gpurun_out/ab_cold_$v.json
  for w in cfg2 cold; do
    echo "v=$v $w $(python -c "import json; d=json.load(open('gpurun_out/ab_${w}_$v.json')); print(round(d['value']/1e6,1), round(d['roofline']['achieved']), round(d['roofline']['frac'],3))")"
  done
done
done
