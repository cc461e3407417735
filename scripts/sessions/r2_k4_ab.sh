#!/bin/bash
# round-2 session: K4 A/B on cfg2 (bulk 1-D copies = variant 2, TMA gather4 =
# variant 3, ALU f32->f64 widening build), gather4 parity, cfg2 cold control,
# ncu of the cfg3 step's K4 (no graph, so the kernel is filterable) and of the
# gather4 kernel.
O=gpurun_out/s2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_g4.py tests/test_gpu_core.py -q -x -p no:cacheprovider > $O/pytest_g4.log 2>&1; echo "rc=$?" >> $O/pytest_g4.log
for rep in 1 2; do
for v in 2 3; do
  FX_POOL_VARIANT=$v timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e > $O/cfg2_v${v}_r$rep.json 2>> $O/bench.err
  FX_POOL_VARIANT=$v timeout 300 python bench.py --config cfg2 --alpha 0 --steps 50 --warmup 5 --no-cpu --no-e2e > $O/cfg2cold_v${v}_r$rep.json 2>> $O/bench.err
done
FX_LIB_PATH=paper_2410_12794_b200/libflexemb_f2d.so timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e > $O/cfg2_f2d_r$rep.json 2>> $O/bench.err
done
FX_POOL_VARIANT=3 timeout 300 python bench.py --steps 40 --warmup 6 --no-cpu --no-e2e > $O/cfg3_v3.json 2>> $O/bench.err
for v in 2 3; do
FX_POOL_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pool -s 3 -c 1 -o $O/k4_cfg2_v$v python bench.py --config cfg2 --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_cfg2_v$v.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pool -s 5 -c 1 -o $O/k4_cfg3 python bench.py --graph-step 0 --steps 2 --warmup 4 --no-cpu --no-e2e > $O/ncu_cfg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --graph-step 0 --steps 2 --warmup 4 --no-cpu --no-e2e > $O/ncu_launch_cfg3.log 2>&1
echo done
