#!/bin/bash
# step parity + timeline + ncu source-level captures of the top step kernels
O=gpurun_out/s4
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_ranker.py -q -x -p no:cacheprovider > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
timeout 400 python scripts/timeline.py --alpha 1.0 --cache 0.02 --steps 4 > $O/tl_1.0_0.02.json 2> $O/tl_1.0_0.02.err
timeout 300 python bench.py --steps 60 --warmup 8 --no-cpu --no-e2e > $O/bench.json 2> $O/bench.err
for k in ks_probe ks_dedup_occ ks_copy_rows ks_apply ks_victim_est ks_age; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o $O/$k python bench.py --graph-step 0 --steps 4 --warmup 8 --no-cpu --no-e2e > $O/ncu_$k.log 2>&1
done
echo done
