#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "rerank or seg or kat or contextual" > gpurun_out/gpu_tests_v.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_v.txt
PROBE_VARIANTS=default,no_net timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_v.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_v.txt
PROBE_SHAPES=148:200:768:10,148:200:768:32,256:200:768:20,148:16:768:10 PROBE_VARIANTS=default,no_net timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_v2.txt 2>&1; echo "rerank2 rc=$?"; cat gpurun_out/rerank_v2.txt
