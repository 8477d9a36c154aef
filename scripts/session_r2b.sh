#!/bin/bash
# Round-2 GPU session b: GPU suite, sanitizers on the extended workload, K3 ncu captures.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_b.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_b.txt
: > gpurun_out/sanitizer_r2.txt
for tool in memcheck racecheck synccheck initcheck; do
  echo "## --tool $tool" >> gpurun_out/sanitizer_r2.txt
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py >> gpurun_out/sanitizer_r2.txt 2>&1; echo "$tool rc=$?"
done
grep -E "^## |SUMMARY|Error|done" gpurun_out/sanitizer_r2.txt | head -30
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rerank -s 3 -c 2 -o gpurun_out/rerank_c3 python scripts/rerank_ncu.py > gpurun_out/rerank_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/rerank_ncu.log
