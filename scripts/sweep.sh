#!/bin/bash
# usage: sweep.sh "rows dim batch [extra...]" ...   (prints ms/step and scan GB/s per case)
for c in "$@"; do
  set -- $c
  r=$1; d=$2; b=$3; shift 3
  timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --rows $r --dim $d --batch $b "$@" \
   | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c', round(d['ms_per_step'],4), round(d['value']), round(d['roofline']['achieved']), round(d['roofline'].get('scan_ms_per_step',0),4))"
done
