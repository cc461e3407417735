#!/bin/bash
# shifted requester order in the owners' gather: parity + cfg4r / cfg5 at N
O=gpurun_out/rot$1
mkdir -p $O
N=$(python -c "import torch; print(torch.cuda.device_count())")
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611"
timeout 1500 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider > $O/pytest_sharded.log 2>&1; echo "rc=$?" >> $O/pytest_sharded.log
timeout 600 $R bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e > $O/bench_cfg4r.json 2> $O/bench_cfg4r.err
timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --config cfg5 --mode rowwise --no-cpu --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 $R bench.py --gpus $N --steps 20 --warmup 3 --config cfg5 --mode rowwise --no-cpu --no-e2e --partial f64 > $O/bench_cfg5_f64.json 2> $O/bench_cfg5_f64.err
echo done
