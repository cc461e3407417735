cd /root/repo
for rep in 1 2; do for cr in 16 12 8; do
  FX_POOL_CR=$cr python bench.py --config cfg1 --graph 64 --steps 640 --warmup 64 --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/d64cr_$cr.json
  echo "cr=$cr $(python -c "import json; d=json.load(open('gpurun_out/d64cr_$cr.json')); print(round(d['value']/1e6,1))")"
done; done
