#!/bin/bash
# real-time kernel timelines (torch.profiler / CUPTI) of the graph-replayed
# cfg3 Ranker batch at three (alpha, cache) points
O=gpurun_out/s3
mkdir -p $O
for ac in "1.0 0.02" "0.6 0.01" "1.2 0.01"; do
  set -- $ac
  timeout 400 python scripts/timeline.py --alpha $1 --cache $2 --steps 4 > $O/tl_$1_$2.json 2> $O/tl_$1_$2.err
done
echo done
