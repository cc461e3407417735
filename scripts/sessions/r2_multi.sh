#!/bin/bash
# multi-GPU evidence for this round's code: sharded parity tests (2 or 4 GPUs),
# the N-GPU bench (cfg4r table-wise default, cfg5 row-wise), reference arm at N
O=gpurun_out/m$1${2:-}
mkdir -p $O
N=$(python -c "import torch; print(torch.cuda.device_count())")
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider > $O/pytest_sharded.log 2>&1; echo "rc=$?" >> $O/pytest_sharded.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $R scripts/comm_check.py > $O/comm_check.log 2>&1; echo "rc=$?" >> $O/comm_check.log
timeout 600 $R bench.py --gpus $N --steps 50 --warmup 5 --no-cpu > $O/bench_cfg4r.json 2> $O/bench_cfg4r.err
timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --config cfg5 --mode rowwise --no-cpu > $O/bench_cfg5.json 2> $O/bench_cfg5.err
for w in cfg4r cfg5 cfg5thr; do
  timeout 600 $R scripts/sharded_bigcheck.py $w --bags 2000 --steps 3 >> $O/bigcheck.jsonl 2>> $O/bigcheck.err; echo "$w rc=$?" >> $O/bigcheck.err
done
echo done
