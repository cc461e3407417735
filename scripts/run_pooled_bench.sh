#!/bin/bash
# pooled-result keyspace cost/benefit at cfg3 scale (32 x 10M x 128)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pooled in 0 1; do
  python scripts/bench_cache.py --alphas 0.8,1.2 --cache-pct 1 --batches 4 --warm 3 --pooled $pooled \
    >> gpurun_out/pooled_bench.jsonl 2>> gpurun_out/pooled_bench.err
  python scripts/bench_cache.py --alphas 1.2 --cache-pct 1 --batches 4 --warm 3 --pooled $pooled --pooling 1,3 \
    --threshold 2 >> gpurun_out/pooled_bench.jsonl 2>> gpurun_out/pooled_bench.err
done
