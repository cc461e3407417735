set -x
nvidia-smi topo -m > gpurun_out/topo9.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_sharded9.log 2>&1
for n in 2 4; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n"
timeout 300 $R bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/b9_n${n}_p2p.log 2>&1
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
timeout 300 $R bench.py --gpus 4 --steps 20 --warmup 3 --mode rowwise --no-e2e > gpurun_out/b9_n4_p2p_row.log 2>&1
timeout 300 $R bench.py --gpus 4 --steps 20 --warmup 3 --exchange nccl --no-e2e > gpurun_out/b9_n4_nccl.log 2>&1
echo done
