#!/bin/bash
# 2 ranks folded onto one GPU: the fused exchange over same-device IPC mappings
O=gpurun_out/s14
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider -k folded > $O/pytest_fold.log 2>&1; echo "rc=$?" >> $O/pytest_fold.log
FX_FOLD_DEVICES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29599 scripts/sharded_check.py rowwise p2pthr > $O/fold_rw_thr.log 2>&1; echo "rc=$?" >> $O/fold_rw_thr.log
echo done
