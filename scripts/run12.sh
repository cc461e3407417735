set -x
timeout 900 python -m pytest tests/test_gpu_cache.py tests/test_gpu_ranker.py -x -q > gpurun_out/p12_cache.log 2>&1
timeout 900 python scripts/bench_cache.py --rows 2000000 --alphas 0.6,1.0,1.2 --cache-pct 1,5 --batches 3 --warm 2 > gpurun_out/b12_cache.log 2>&1
echo done
