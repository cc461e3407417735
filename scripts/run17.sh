set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/p17_all.log 2>&1
python bench.py > gpurun_out/b17_full.log 2>&1
python bench.py --config cfg1 --steps 640 --warmup 10 --no-cpu --no-e2e > gpurun_out/b17_cfg1.log 2>&1
python bench.py --config cfg1 --graph 64 --steps 640 --warmup 10 --no-cpu --no-e2e > gpurun_out/b17_cfg1_graph.log 2>&1
python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/b17_cold.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain17a.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches17.csv $B > gpurun_out/ncu17a.log 2>&1
$B > gpurun_out/plain17b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pool_async -s 4 -c 1 -o gpurun_out/prof17 $B > gpurun_out/ncu17b.log 2>&1
$B --alpha 0 --table-rows 4000000 > gpurun_out/plain17c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pool_async -s 4 -c 1 -o gpurun_out/prof17_cold $B --alpha 0 --table-rows 4000000 > gpurun_out/ncu17c.log 2>&1
timeout 1500 python scripts/bench_cache.py --rows 10000000 --alphas 0.6,0.8,1.0,1.2 --cache-pct 1,2 --batches 3 --warm 2 > gpurun_out/b17_cache_full.log 2>&1
echo done
