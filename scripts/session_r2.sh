#!/bin/bash
# Round-2 standard GPU session: tests, smoke, bench, rerank probe, launch list.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_default.json
timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_probe.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/rerank_probe.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
python profiles/launch_summary.py gpurun_out/launches_r2.csv 20 2>&1 | tail -25
