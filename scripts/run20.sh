set -x
timeout 900 python -m pytest tests/test_gpu_cache.py tests/test_gpu_ranker.py -x -q > gpurun_out/p20_cache.log 2>&1
FX_CACHE_PROFILE=1 timeout 900 python scripts/bench_cache.py --rows 10000000 --alphas 0.6,1.0 --cache-pct 1,2 --batches 2 --warm 2 > gpurun_out/b20_cache.log 2> gpurun_out/b20_cache_prof.log
timeout 1500 python scripts/bench_cache.py --rows 10000000 --alphas 0.6,0.8,1.0,1.2 --cache-pct 1,2 --batches 3 --warm 2 > gpurun_out/b20_cache_full.log 2>&1
echo done
