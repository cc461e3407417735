#!/bin/bash
# N=2 A/B of the pipelined stage (push) against the concurrent gather:
# push grid blocks/SM (FX_PUSH_BPS) and the non-pipelined (--sync) control.
cd "$(dirname "$0")/.."; mkdir -p gpurun_out
run() { timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 --no-e2e --no-cpu --steps 300 $2 2>/dev/null | tail -1 > gpurun_out/ab_$3.json; echo "$3 $(python -c "import json; d=json.load(open('gpurun_out/ab_$3.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],4), d['roofline']['pool_ms_per_step_all_ranks'], d['a2a']['phases_ms_total'])")"; }
for rep in 1 2; do
for v in 1 0; do for b in 1 8; do FX_PUSH_VALIDATE=$v FX_PUSH_BPS=$b run 296$v$b "" v${v}bps$b; done; done
done
