#!/bin/bash
# one GPU, shard-sized corpora of the N=2/4/8 split (10M/N rows, B=1024, k=10): the per-rank scan
# a sharded run would do (no exchange; K6 measured separately by scripts/k6_probe.py)
set -u
mkdir -p gpurun_out
for n in 5000000 2500000 1250000; do
  timeout 600 python bench.py --rows $n --no-cpu-baseline > gpurun_out/bench_shard_$n.json 2>&1; echo "rows $n rc=$?"
  python -c "
import json
l=[x for x in open('gpurun_out/bench_shard_$n.json').read().splitlines() if x.startswith('{')][-1]; d=json.loads(l)
print($n, round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
