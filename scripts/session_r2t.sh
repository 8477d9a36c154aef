#!/bin/bash
set -u
mkdir -p gpurun_out
PROBE_PROFILE=b200 PROBE_ISOLATED=1 timeout 900 python scripts/stream_probe.py > gpurun_out/stream_iso_b200.jsonl 2>&1; echo "iso b200 rc=$?"; cat gpurun_out/stream_iso_b200.jsonl
PROBE_PROFILE=b200 timeout 900 python scripts/stream_probe.py > gpurun_out/stream_b200.jsonl 2>&1; echo "b200 rc=$?"; cat gpurun_out/stream_b200.jsonl
