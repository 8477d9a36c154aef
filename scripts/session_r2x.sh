#!/bin/bash
# final-tree re-check after the K3 top-k network: full GPU suite + smoke + default bench
set -u
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_x.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_x.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_x.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_x.txt
timeout 900 python bench.py > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err; echo "bench rc=$?"; tail -c 250 gpurun_out/bench_x.json
