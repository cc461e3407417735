set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/p16_sharded.log 2>&1
for n in 2 4; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n"
timeout 300 $R bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/b16_n${n}_tw.log 2>&1
timeout 300 $R bench.py --gpus $n --steps 30 --warmup 3 --no-e2e --mode rowwise > gpurun_out/b16_n${n}_rw.log 2>&1
timeout 300 $R bench.py --gpus $n --steps 30 --warmup 3 --no-e2e --mode rowwise --partial f32 > gpurun_out/b16_n${n}_rw32.log 2>&1
timeout 300 $R bench.py --gpus $n --steps 50 --warmup 5 --no-e2e --replicate-rows 1000000 > gpurun_out/b16_n${n}_hyb.log 2>&1
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711"
timeout 900 $R bench.py --gpus 4 --config cfg5 --mode rowwise --partial f32 --batches 2 --steps 10 --warmup 2 --no-e2e > gpurun_out/b16_n4_cfg5_f32.log 2>&1
timeout 900 $R bench.py --gpus 4 --config cfg4r --batches 2 --steps 30 --warmup 3 --no-e2e > gpurun_out/b16_n4_cfg4r.log 2>&1
echo done
