set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest8.log 2>&1
python bench.py > gpurun_out/b8_full.log 2>&1
python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b8_cold.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches8.csv $B > gpurun_out/ncu8a.log 2>&1
$B > gpurun_out/plain8b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pool_async -s 4 -c 1 -o gpurun_out/prof8_async $B > gpurun_out/ncu8b.log 2>&1
$B --alpha 0 --table-rows 4000000 > gpurun_out/plain8c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pool_async -s 4 -c 1 -o gpurun_out/prof8_async_cold $B --alpha 0 --table-rows 4000000 > gpurun_out/ncu8c.log 2>&1
echo done
