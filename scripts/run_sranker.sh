#!/bin/bash
cd "$(dirname "$0")/.."
N=${N:-2}
i=0
for a in "2" "none" "2 pooled" "none pooled"; do
  i=$((i+1))
  torchrun --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969$i scripts/sharded_ranker_check.py $a \
    > gpurun_out/sranker_$i.log 2>&1
  echo "rc=$? $(grep SHARDED_RANKER gpurun_out/sranker_$i.log)"
done
