#!/bin/bash
# hard-victim bitmap + identity offer list (one batch in flight): parity + A/B
O=gpurun_out/s19
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_ranker.py tests/test_gpu_cache.py tests/test_gpu_pooled.py tests/test_gpu_integration.py -q -x -p no:cacheprovider > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
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
