#!/bin/bash
# both arms as the driver launches them, N=1 and N=4: identical config dicts
O=gpurun_out/dcfg
mkdir -p $O
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/ref1.json 2> $O/ref1.err
timeout 900 python bench.py --steps 40 --warmup 5 --no-cpu > $O/ours1.json 2> $O/ours1.err
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641"
timeout 900 $R bench.py --impl reference --gpus 4 --steps 5 --warmup 3 > $O/ref4.json 2> $O/ref4.err
timeout 900 $R bench.py --gpus 4 --steps 50 --warmup 5 > $O/ours4.json 2> $O/ours4.err
echo done
