#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_backend.py tests/test_gpu_launcher.py tests/test_gpu_sharded_index.py -x -q > gpurun_out/gpu_tests_u.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_u.txt
PROBE_PROFILE=b200 PROBE_ISOLATED=1 timeout 900 python scripts/stream_probe.py > gpurun_out/stream_u1.jsonl 2>&1; echo "iso b200 rc=$?"; cat gpurun_out/stream_u1.jsonl
PROBE_PROFILE=b200 timeout 900 python scripts/stream_probe.py > gpurun_out/stream_u2.jsonl 2>&1; echo "b200 rc=$?"; cat gpurun_out/stream_u2.jsonl
timeout 900 python scripts/stream_probe.py > gpurun_out/stream_u3.jsonl 2>&1; echo "ref rc=$?"; cat gpurun_out/stream_u3.jsonl
