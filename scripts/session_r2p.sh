#!/bin/bash
# paired-ring identity test; K3 per-SM balance diagnostic (1 vs 2 blocks per SM at C3's row size)
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_search.py -x -q -k "paired or ring_equals" > gpurun_out/gpu_tests_p.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_p.txt
PROBE_SHAPES=148:200:768:10,200:200:768:10,256:200:768:10,296:200:768:10,444:200:768:10 PROBE_VARIANTS=ring_s2,ring_s4 timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_p.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_p.txt
