set -x
nproc > gpurun_out/nproc.txt
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_pool -s 4 -c 1 -o gpurun_out/prof_pool $B > gpurun_out/ncu_full.log 2>&1
$B --alpha 0 > gpurun_out/plain_cold.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_pool -s 4 -c 1 -o gpurun_out/prof_pool_cold $B --alpha 0 > gpurun_out/ncu_full_cold.log 2>&1
python bench.py --steps 200 --warmup 10 --alpha 0 --no-cpu > gpurun_out/bench_cold.log 2>&1
python bench.py > gpurun_out/bench_full.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo done
