#!/bin/bash
# Round-2 closing session on the final tree: full GPU suite, smoke, default bench (our arm and
# the reference arm), k=100, C2 shape, fp32 mode, 200-step stability run, launch list, full
# ncu of the headline kernel, per-kernel table, primitives, K6 probe, workflows.
set -u
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_z.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_z.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_z.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_z.txt
timeout 900 python bench.py > gpurun_out/bench_z.json 2> gpurun_out/bench_z.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_z.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_z.json 2> gpurun_out/bench_ref_z.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref_z.json
timeout 900 python bench.py --k 100 --no-cpu-baseline > gpurun_out/bench_k100_z.json 2>&1; echo "k100 rc=$?"
timeout 900 python bench.py --rows 1000000 --dim 768 --batch 256 --no-cpu-baseline > gpurun_out/bench_c2_z.json 2>&1; echo "c2 rc=$?"
timeout 900 python bench.py --rows 1000000 --storage f32 --no-cpu-baseline > gpurun_out/bench_f32_z.json 2>&1; echo "f32 rc=$?"
timeout 900 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/bench_200_z.json 2>&1; echo "200 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_z.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_topk_pair -s 6 -c 1 -o gpurun_out/headline_z python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/ktable_z.csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed python scripts/kernel_table.py > gpurun_out/ktable_z_run.log 2>&1; echo "ktable rc=$?"
python scripts/kernel_table.py --summarize gpurun_out/ktable_z.csv > gpurun_out/ktable_z.txt 2>&1
timeout 600 python bench_primitives.py > gpurun_out/prims_z.jsonl 2> gpurun_out/prims_z.err; echo "prims rc=$?"
timeout 600 python scripts/k6_probe.py > gpurun_out/k6_z.txt 2>&1; echo "k6 rc=$?"
PROBE_VARIANTS=default timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_z.txt 2>&1; echo "rerank rc=$?"
timeout 1500 python bench_workflows.py > gpurun_out/workflows_z.jsonl 2>&1; echo "wf rc=$?"
