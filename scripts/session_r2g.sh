#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_g.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_g.txt; grep -E "^FAILED|Error" gpurun_out/pytest_g.txt | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
: > gpurun_out/sanitizer_g.txt
for tool in memcheck racecheck synccheck; do
  echo "## --tool $tool" >> gpurun_out/sanitizer_g.txt
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py >> gpurun_out/sanitizer_g.txt 2>&1; echo "$tool rc=$?"
done
grep -E "^## |SUMMARY|done" gpurun_out/sanitizer_g.txt | head -20
timeout 600 python bench_primitives.py > gpurun_out/prims_g.jsonl 2>gpurun_out/prims_g.err; echo "prims rc=$?"
