#!/bin/bash
# world size 8 folded onto the box's GPUs (2 ranks per GPU on a 4-GPU box):
# the exchange protocol at N=8 (IPC windows, 8-way barrier, shifted order)
O=gpurun_out/w8
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29631"
for me in "tablewise p2p" "rowwise p2p" "rowwise p2pthr" "tablewise p2p-pipe" "rowwise p2p-pipe"; do
  set -- $me
  FX_FOLD_DEVICES=1 timeout 600 $R scripts/sharded_check.py $1 $2 >> $O/w8.log 2>&1; echo "$1 $2 rc=$?" >> $O/w8.log
done
FX_FOLD_DEVICES=1 timeout 600 $R scripts/sharded_ranker_check.py 2 >> $O/w8.log 2>&1; echo "sranker rc=$?" >> $O/w8.log
echo done
