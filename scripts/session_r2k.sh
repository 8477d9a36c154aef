#!/bin/bash
# K3 lists kernel without the early PDL trigger (A/B against session j), ring default.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "rerank or seg or kat or small or contextual or merge" > gpurun_out/gpu_tests_k.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_k.txt
PROBE_VARIANTS=default,lists,lists_s3 timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_k.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_k.txt
PROBE_SHAPES=1024:50:768:10,512:100:1024:10 PROBE_VARIANTS=default,lists timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_k2.txt 2>&1; echo "rerank2 rc=$?"; cat gpurun_out/rerank_k2.txt
