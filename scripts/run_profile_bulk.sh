#!/bin/bash
# correctness + ncu evidence for the default K4 (TMA bulk-copy staging)
cd "$(dirname "$0")/.."
python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/pb_bench.json 2>gpurun_out/pb_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_bulk.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/pb_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pool_bulk -s 5 -c 1 -o gpurun_out/prof_bulk_cfg2 \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/pb_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pool_bulk -s 5 -c 1 -o gpurun_out/prof_bulk_cold \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --alpha 0 --table-rows 4000000 > gpurun_out/pb_ncu3.log 2>&1
ls -la gpurun_out/prof_bulk_* gpurun_out/r1_launches_bulk.csv
