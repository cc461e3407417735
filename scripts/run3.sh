set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1
for v in 0 1 2; do
  FX_POOL_VARIANT=$v python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e > gpurun_out/b3_v$v.log 2>&1
  FX_POOL_VARIANT=$v python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b3_cold_v$v.log 2>&1
done
echo done
