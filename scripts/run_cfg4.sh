#!/bin/bash
# cfg4 (DLRM-RM2 100 x 10M x 128, table-wise) and its row-reduced 1->2->4 curve (cfg4r, 100 x 1M)
cd "$(dirname "$0")/.."
python bench.py --config cfg4r --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/c4r_1.json
for n in 2 4; do
  torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2980$n bench.py --gpus $n --config cfg4r \
    --steps 50 --warmup 5 --no-e2e --replicate-rows 0 2>/dev/null | tail -1 > gpurun_out/c4r_$n.json
done
torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29809 bench.py --gpus 4 --config cfg4 \
  --steps 30 --warmup 5 --no-e2e --replicate-rows 0 2>/dev/null | tail -1 > gpurun_out/c4_4.json
for f in c4r_1 c4r_2 c4r_4 c4_4; do
  echo "$f $(python -c "import json; d=json.load(open('gpurun_out/$f.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), d['config'].get('parallelism'), d['roofline'].get('frac'))")"
done
