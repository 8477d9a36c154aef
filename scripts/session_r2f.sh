#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -x -k "small_scan or search_matches or ties or identity or k_exceeds or planted" > gpurun_out/pytest_f.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_f.txt
timeout 600 python bench_primitives.py --configs c1 > gpurun_out/prims_f.jsonl 2>gpurun_out/prims_f.err; echo "prims rc=$?"; cut -c1-300 gpurun_out/prims_f.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:small_scan -c 3 python bench_primitives.py --configs c1 --reps 2 2>&1 | grep -E "duration|inst_exec" | head -6
