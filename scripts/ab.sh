#!/bin/bash
# usage: ab.sh "ENV=.. ENV2=.." "ENV=.." ... -- bench args : A/B the bench under env settings,
# interleaved twice; prints ms/step, q/s, roofline frac and median SM clock per run.
cfgs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do cfgs+=("$1"); shift; done; shift
for rep in 1 2; do for c in "${cfgs[@]}"; do
  env $c timeout 300 python bench.py --no-cpu-baseline "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c'.ljust(40), round(d['ms_per_step'],3), int(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done
