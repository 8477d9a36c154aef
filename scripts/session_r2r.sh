#!/bin/bash
# K3 selection with pre-sorted lane heads: parity subset + fixed-cost probe + C3 / C5 shapes
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "rerank or seg or kat or contextual or merge" > gpurun_out/gpu_tests_r.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_r.txt
PROBE_SHAPES=148:16:768:1,148:16:768:10,148:200:768:1,148:200:768:10,1:200:768:10,256:200:768:10,16:32:1024:3,256:200:1024:10,256:400:768:40 PROBE_VARIANTS=default timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_r.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_r.txt
timeout 600 python bench_primitives.py > gpurun_out/prims_r.jsonl 2> gpurun_out/prims_r.err; echo "prims rc=$?"; grep -o '"config": "C[15][^"]*"\|"device_ms_cuda_graph": [0-9.]*\|"fused_chain_ms_cuda_graph": [0-9.]*' gpurun_out/prims_r.jsonl
