#!/bin/bash
# compute-sanitizer on the late round-2 tree (paired K3 ring, redux selection, early PDL trigger).
set -u
mkdir -p gpurun_out
out=gpurun_out/sanitizer_late.txt
echo "# compute-sanitizer on the late round-2 tree (scripts/sanitize.py: K1 / K2t / K2s / fused C5 / K3 ring s2 + paired s4 / lists / sort / split)" > $out
for tool in memcheck synccheck initcheck racecheck; do
  echo "## --tool $tool" >> $out
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py >> $out 2>&1; echo "$tool rc=$?"
done
grep -c "Race reported" $out; grep "ERROR SUMMARY" $out
