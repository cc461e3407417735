set -x
for cr in 16 12 8; do
  FX_POOL_CR=$cr python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e > gpurun_out/b14_cr$cr.log 2>&1
  FX_POOL_CR=$cr python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b14_cold_cr$cr.log 2>&1
  FX_LIB_PATH=paper_2410_12794_b200/libflexemb_minb6.so FX_POOL_CR=$cr python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e > gpurun_out/b14m6_cr$cr.log 2>&1
  FX_LIB_PATH=paper_2410_12794_b200/libflexemb_minb6.so FX_POOL_CR=$cr python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b14m6_cold_cr$cr.log 2>&1
done
FX_POOL_CR=8 timeout 600 python -m pytest tests/test_gpu_core.py -x -q > gpurun_out/p14_cr8.log 2>&1
echo done
