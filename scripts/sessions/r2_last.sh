#!/bin/bash
# last check of the final tree: the bench-contract GPU test, both arms at N=1 with the driver's flags
O=gpurun_out/last
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bench or smoke or folded" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/ref1.json 2> $O/ref1.err
timeout 900 python bench.py --steps 20 --warmup 3 > $O/ours1.json 2> $O/ours1.err
echo done
