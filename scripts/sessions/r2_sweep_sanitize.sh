#!/bin/bash
# round-2 session: cfg3 alpha sweep (bench.py, graph-replayed Ranker batch),
# compute-sanitizer over the fused step and the single-GPU kernels, and one
# ncu --set full capture of K4 inside the cfg3 bench (DRAM traffic).
mkdir -p gpurun_out/s1
O=gpurun_out/s1
for a in 0.6 0.8 1.0 1.2; do for c in 0.01 0.02; do
  timeout 300 python bench.py --alpha $a --cache $c --steps 40 --warmup 6 --no-cpu --no-e2e >> $O/sweep.jsonl 2>> $O/sweep.err
done; done
CS=/usr/local/cuda/bin/compute-sanitizer
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $t --print-limit 50 python scripts/sanitize_step.py > $O/san_step_$t.log 2>&1; echo "rc=$?" >> $O/san_step_$t.log
done
timeout 1200 $CS --tool memcheck --print-limit 50 python -m pytest tests -m gpu -x -q -k "core or cache or pooled" -p no:cacheprovider > $O/san_pytest_memcheck.log 2>&1; echo "rc=$?" >> $O/san_pytest_memcheck.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pool_bulk -s 12 -c 1 -o $O/k4_cfg3 python bench.py --steps 2 --warmup 4 --no-cpu --no-e2e > $O/ncu_k4.log 2>&1
echo done
