#!/bin/bash
# K3 rerank: redux.sync warp selection + early PDL trigger. Parity subset, probe, ncu of K3 at C3.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "rerank or seg or kat or small or contextual or merge" > gpurun_out/gpu_tests_j.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_j.txt
PROBE_VARIANTS=default,lists,sort_s2 timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_j.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_j.txt
PROBE_VARIANTS=default timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_j2.txt 2>&1; echo "rerank2 rc=$?"; cat gpurun_out/rerank_j2.txt
timeout 600 python bench_primitives.py > gpurun_out/prims_j.jsonl 2> gpurun_out/prims_j.err; echo "prims rc=$?"; cat gpurun_out/prims_j.jsonl | cut -c1-400
