#!/bin/bash
# side-stream row copies: parity + A/B + timeline
O=gpurun_out/s7
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_ranker.py -q -x -p no:cacheprovider > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
for rep in 1 2; do
for cs in 1 0; do
  for a in 1.0 0.6 1.2; do
    c=0.02; [ $a != 1.0 ] && c=0.01
    FX_COPY_SIDE=$cs timeout 300 python bench.py --alpha $a --cache $c --steps 40 --warmup 6 --no-cpu --no-e2e > $O/b_cs${cs}_a${a}_r$rep.json 2>> $O/bench.err
  done
done
done
timeout 400 python scripts/timeline.py --alpha 1.0 --cache 0.02 --steps 4 > $O/tl_1.0_0.02.json 2> $O/tl_1.0_0.02.err
echo done
