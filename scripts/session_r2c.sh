#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -k "rerank" > gpurun_out/pytest_rerank.txt 2>&1; echo "pytest rerank rc=$?"; tail -3 gpurun_out/pytest_rerank.txt
timeout 600 python -m pytest tests/test_gpu_peer.py -m gpu -q > gpurun_out/pytest_peer.txt 2>&1; echo "pytest peer rc=$?"; tail -3 gpurun_out/pytest_peer.txt
timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_probe2.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/rerank_probe2.txt
timeout 600 python scripts/k6_probe.py > gpurun_out/k6_probe.txt 2>&1; echo "k6 rc=$?"; cat gpurun_out/k6_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rerank_mma -s 3 -c 1 -o gpurun_out/rerank_mma_c3 python scripts/rerank_ncu.py > gpurun_out/rerank_ncu2.log 2>&1; echo "ncu rc=$?"
