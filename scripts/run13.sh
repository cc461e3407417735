set -x
for cr in 24 16; do FX_POOL_CR=$cr timeout 600 python -m pytest tests/test_gpu_core.py -x -q > gpurun_out/p13_cr$cr.log 2>&1; done
for cr in 32 24 16; do
  FX_POOL_CR=$cr python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e > gpurun_out/b13_cr$cr.log 2>&1
  FX_POOL_CR=$cr python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b13_cold_cr$cr.log 2>&1
done
echo done
