#!/bin/bash
# Round-2 late refresh after the K3 selection / routing and host-path changes: full GPU suite,
# smoke, per-kernel ncu table, primitives, workflow bench, stream probe.
set -u
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_h.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_h.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_h.txt
timeout 900 ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/ktable_h.csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed python scripts/kernel_table.py > gpurun_out/ktable_h_run.log 2>&1; echo "ktable rc=$?"
python scripts/kernel_table.py --summarize gpurun_out/ktable_h.csv > gpurun_out/ktable_h.txt 2>&1; cat gpurun_out/ktable_h.txt
timeout 600 python bench_primitives.py > gpurun_out/prims_h.jsonl 2> gpurun_out/prims_h.err; echo "prims rc=$?"
timeout 1500 python bench_workflows.py > gpurun_out/workflows_h.jsonl 2>&1; echo "wf rc=$?"
timeout 600 python scripts/stream_probe.py > gpurun_out/stream_h.jsonl 2>&1; echo "stream rc=$?"
