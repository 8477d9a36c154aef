#!/bin/bash
# usage: launches.sh tag N "bench args" -> ncu launch list of the last N launches
tag=$1; n=$2; shift 2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/l_$tag.csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 "$@" >/dev/null 2>&1
python profiles/launch_summary.py gpurun_out/l_$tag.csv $n | sed "s/^/$tag /"
