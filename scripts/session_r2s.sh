#!/bin/bash
# bench p2p self-check (ranks sharing one GPU over gloo) + default bench line
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench.py tests/test_gpu_peer.py -x -q > gpurun_out/gpu_tests_s.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s.txt
