#!/bin/bash
# sketch tombstone reuse: parity + long-run bench (200 steps, as the driver runs it)
O=gpurun_out/s15
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_ranker.py tests/test_gpu_cache.py tests/test_gpu_pooled.py -q -x -p no:cacheprovider > $O/pytest_step.log 2>&1; echo "rc=$?" >> $O/pytest_step.log
FX_LIB_PATH=$PWD/paper_2410_12794_b200/libflexemb_chk.so timeout 900 python scripts/sanitize_step.py > $O/sanitize_chk.log 2>&1; echo "rc=$?" >> $O/sanitize_chk.log
timeout 1500 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider -k folded > $O/pytest_fold.log 2>&1; echo "rc=$?" >> $O/pytest_fold.log
for r in 1 2; do
  timeout 600 python bench.py --no-cpu --no-e2e > $O/b200_r$r.json 2>> $O/bench.err
done
for a in 1.0 0.6 1.2; do
  c=0.02; [ $a != 1.0 ] && c=0.01
  timeout 300 python bench.py --alpha $a --cache $c --steps 40 --warmup 6 --no-cpu --no-e2e > $O/b_a${a}.json 2>> $O/bench.err
  timeout 600 python bench.py --alpha $a --cache $c --steps 200 --warmup 10 --no-cpu --no-e2e > $O/b200_a${a}.json 2>> $O/bench.err
done
echo done
