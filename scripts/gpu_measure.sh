#!/bin/bash
# One GPU session of measurements (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
run() { local name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err; echo "$name rc=$?"; tail -c 600 gpurun_out/$name.json; echo; }
run bench_default
run bench_reference --impl reference --steps 3 --warmup 1
run bench_k100 --k 100 --no-cpu-baseline --steps 5 --warmup 3
run bench_c2 --rows 1000000 --dim 768 --batch 256 --no-cpu-baseline --steps 20 --warmup 5
run bench_f32 --storage f32 --no-cpu-baseline --steps 3 --warmup 3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
