set -x
for v in 3 4 5; do FX_POOL_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_core.py -x -q > gpurun_out/p10_v$v.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_ranker.py -x -q > gpurun_out/p10_ranker.log 2>&1
for v in 1 3 4 5; do
  FX_POOL_VARIANT=$v python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e > gpurun_out/b10_v$v.log 2>&1
  FX_POOL_VARIANT=$v python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b10_cold_v$v.log 2>&1
done
timeout 900 python scripts/bench_cache.py --rows 2000000 --alphas 0.6,1.0,1.2 --cache-pct 1,5 --batches 4 --warm 3 > gpurun_out/b10_cache_small.log 2>&1
echo done
