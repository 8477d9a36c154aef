#!/bin/bash
# Host-path changes (host row table for the fused chain, in-edge index): backend / launcher /
# fused-chain GPU tests, stream probe, host profile.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_backend.py tests/test_gpu_launcher.py tests/test_gpu_kats.py -x -q > gpurun_out/gpu_tests_n.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_n.txt
timeout 900 python -m pytest tests/test_gpu_search.py -x -q -k "fused or segmented" > gpurun_out/gpu_tests_n2.txt 2>&1; echo "tests2 rc=$?"; tail -1 gpurun_out/gpu_tests_n2.txt
timeout 600 python scripts/stream_probe.py > gpurun_out/stream_n.jsonl 2>&1; echo "stream rc=$?"; cat gpurun_out/stream_n.jsonl
timeout 600 python scripts/host_profile.py > gpurun_out/host_profile_n.txt 2>&1; echo "hostprof rc=$?"; grep -E "backend|index|_native" gpurun_out/host_profile_n.txt | head -40
