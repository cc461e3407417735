#!/bin/bash
# sketch age from the live-flag bytes: full GPU suite + bounds build + A/B
O=gpurun_out/s20
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
FX_LIB_PATH=$PWD/paper_2410_12794_b200/libflexemb_chk.so timeout 900 python scripts/sanitize_step.py > $O/sanitize_chk.log 2>&1; echo "rc=$?" >> $O/sanitize_chk.log
for r in 1 2; do
  for a in 1.0 0.6 1.2; do
    c=0.02; [ $a != 1.0 ] && c=0.01
    timeout 300 python bench.py --alpha $a --cache $c --steps 40 --warmup 6 --no-cpu --no-e2e > $O/b_a${a}_r$r.json 2>> $O/bench.err
  done
done
timeout 600 python bench.py --no-cpu --no-e2e > $O/b200.json 2>> $O/bench.err
timeout 400 python scripts/timeline.py --alpha 1.0 --cache 0.02 --steps 4 > $O/tl_1.0_0.02.json 2> $O/tl_1.0_0.02.err
echo done
