#!/bin/bash
# Round-2 re-entry check on the restored tree: full GPU suite, smoke, default bench.
set -u
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_i.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_i.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_i.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_i.txt
timeout 900 python bench.py > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_i.json
timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_i.txt 2>&1; echo "rerank rc=$?"; tail -20 gpurun_out/rerank_i.txt
