set -x
timeout 1200 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/p21_sharded.log 2>&1
for n in 2 4; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n"
timeout 300 $R bench.py --gpus $n --no-e2e > gpurun_out/b21_n${n}_pipe.log 2>&1
timeout 300 $R bench.py --gpus $n --no-e2e --sync > gpurun_out/b21_n${n}_sync.log 2>&1
FX_POOL_MAXB=5 timeout 300 $R bench.py --gpus $n --no-e2e > gpurun_out/b21_n${n}_pipe_maxb5.log 2>&1
timeout 300 $R bench.py --gpus $n --no-e2e --replicate-rows 0 > gpurun_out/b21_n${n}_pipe_tw.log 2>&1
done
echo done
