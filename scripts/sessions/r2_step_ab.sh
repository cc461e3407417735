#!/bin/bash
# step parity after the probe / dedup changes + dedup bags-per-warp A/B + timeline
O=gpurun_out/s6
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_ranker.py tests/test_gpu_cache.py -q -x -p no:cacheprovider > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
for bw in 8 32 4 16; do
  for a in 1.0 0.6 1.2; do
    c=0.02; [ $a != 1.0 ] && c=0.01
    FX_DEDUP_BW=$bw timeout 300 python bench.py --alpha $a --cache $c --steps 40 --warmup 6 --no-cpu --no-e2e > $O/b_bw${bw}_a$a.json 2>> $O/bench.err
  done
done
timeout 400 python scripts/timeline.py --alpha 1.0 --cache 0.02 --steps 4 > $O/tl_1.0_0.02.json 2> $O/tl_1.0_0.02.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ks_probe -s 8 -c 1 -o $O/ks_probe python bench.py --graph-step 0 --steps 4 --warmup 8 --no-cpu --no-e2e > $O/ncu_ks_probe.log 2>&1
echo done
