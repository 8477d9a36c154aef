#!/bin/bash
# Round-2 closing measurements: bench, launch list, full ncu of the headline kernel, per-kernel
# table, primitives, K6 probe, workflow bench.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"; tail -c 700 gpurun_out/bench_final.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_topk_pair -s 6 -c 1 -o gpurun_out/headline_r2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/ktable_r2.csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed python scripts/kernel_table.py > gpurun_out/ktable_run.log 2>&1; echo "ktable rc=$?"
python scripts/kernel_table.py --summarize gpurun_out/ktable_r2.csv > gpurun_out/ktable_r2.txt 2>&1; cat gpurun_out/ktable_r2.txt
timeout 600 python bench_primitives.py > gpurun_out/prims_final.jsonl 2> gpurun_out/prims_final.err; echo "prims rc=$?"
timeout 600 python scripts/k6_probe.py > gpurun_out/k6_final.txt 2>&1; echo "k6 rc=$?"
timeout 1500 python bench_workflows.py > gpurun_out/workflows_final.jsonl 2>&1; echo "wf rc=$?"
timeout 600 python scripts/stream_probe.py > gpurun_out/stream_final.jsonl 2>&1; echo "stream rc=$?"
