#!/bin/bash
# probe keys-in-flight A/B (2 vs 4) + parity under 4
O=gpurun_out/s16
mkdir -p $O
FX_PROBE_ILP=4 timeout 900 python -m pytest tests/test_gpu_step.py -q -x -p no:cacheprovider > $O/pytest_step4.log 2>&1; echo "rc=$?" >> $O/pytest_step4.log
for r in 1 2; do for ilp in 2 4; do
  for a in 1.0 0.6 1.2; do
    c=0.02; [ $a != 1.0 ] && c=0.01
    FX_PROBE_ILP=$ilp timeout 300 python bench.py --alpha $a --cache $c --steps 40 --warmup 6 --no-cpu --no-e2e > $O/b_ilp${ilp}_a${a}_r$r.json 2>> $O/bench.err
  done
done; done
echo done
