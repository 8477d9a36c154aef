#!/bin/bash
# K3 fixed-cost decomposition: tiny candidate lists, k=1 vs k=10, 1 vs 200 candidates
set -u
mkdir -p gpurun_out
PROBE_SHAPES=148:16:768:1,148:16:768:10,148:64:768:10,148:200:768:1,148:200:768:10,1:200:768:10,16:200:768:10,296:16:768:10 PROBE_VARIANTS=ring_s2 timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_q.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_q.txt
