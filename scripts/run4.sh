set -x
FX_POOL_VARIANT=1 python -m pytest tests/test_gpu_core.py -x -q > gpurun_out/pytest_v1.log 2>&1
FX_POOL_VARIANT=2 python -m pytest tests/test_gpu_core.py -x -q > gpurun_out/pytest_v2.log 2>&1
for v in 0 1 2; do
  FX_POOL_VARIANT=$v python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e > gpurun_out/b4_v$v.log 2>&1
  FX_POOL_VARIANT=$v python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b4_cold_v$v.log 2>&1
done
echo done
