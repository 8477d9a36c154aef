#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -x > gpurun_out/pytest_e.txt 2>&1; echo "pytest search rc=$?"; tail -15 gpurun_out/pytest_e.txt
timeout 600 python bench_primitives.py --configs c1,c5 > gpurun_out/prims_e.jsonl 2>gpurun_out/prims_e.err; echo "prims rc=$?"; cut -c1-600 gpurun_out/prims_e.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:small_scan -c 5 python bench_primitives.py --configs c1 --reps 2 2>&1 | grep -E "small_scan|duration" | head -10
