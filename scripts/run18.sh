set -x
for n in 2 4; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2980$n"
timeout 300 $R bench.py --gpus $n > gpurun_out/b18_n${n}_default.log 2>&1
timeout 300 $R bench.py --gpus $n --steps 100 --warmup 5 --no-e2e --replicate-rows 0 > gpurun_out/b18_n${n}_tw.log 2>&1
done
echo done
