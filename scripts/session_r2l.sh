#!/bin/bash
# K3 ring: 4 slots consumed two rows at a time (TSV_RERANK_SLOTS=4) vs 2 slots; parity under both.
set -u
mkdir -p gpurun_out
TSV_RERANK_SLOTS=4 timeout 900 python -m pytest tests -m gpu -x -q -k "rerank or seg or kat or contextual" > gpurun_out/gpu_tests_l4.txt 2>&1; echo "tests s4 rc=$?"; tail -1 gpurun_out/gpu_tests_l4.txt
PROBE_VARIANTS=ring_s2,ring_s3,ring_s4 timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_l.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_l.txt
PROBE_SHAPES=64:100:1024:10,256:50:768:10,128:200:1024:10 PROBE_VARIANTS=ring_s2,ring_s4 timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_l2.txt 2>&1; echo "rerank2 rc=$?"; cat gpurun_out/rerank_l2.txt
PROBE_VARIANTS=ring_s4,ring_s2 timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_l3.txt 2>&1; echo "rerank3 rc=$?"; cat gpurun_out/rerank_l3.txt
