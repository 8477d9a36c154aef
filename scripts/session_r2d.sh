#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_launcher.py tests/test_gpu_peer.py -m gpu -q -x > gpurun_out/pytest_d.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_d.txt
timeout 600 python scripts/k6_probe.py > gpurun_out/k6_probe2.txt 2>&1; echo "k6 rc=$?"; cat gpurun_out/k6_probe2.txt
timeout 600 python bench_primitives.py --configs c1,c5,c3 > gpurun_out/prims_d.jsonl 2>gpurun_out/prims_d.err; echo "prims rc=$?"; cat gpurun_out/prims_d.jsonl | cut -c1-700
