set -x
timeout 600 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded7.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500"
timeout 300 $R bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/b7_n2_p2p.log 2>&1
timeout 300 $R bench.py --gpus 2 --steps 20 --warmup 3 --mode rowwise --no-e2e > gpurun_out/b7_n2_p2p_row.log 2>&1
timeout 300 $R bench.py --gpus 2 --steps 50 --warmup 5 --exchange nccl --no-e2e > gpurun_out/b7_n2_nccl.log 2>&1
echo done
