set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all2.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29500"
$R bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/bench_n2.log 2>&1
$R bench.py --gpus 2 --steps 20 --warmup 3 --mode rowwise --no-e2e > gpurun_out/bench_n2_row.log 2>&1
echo done
