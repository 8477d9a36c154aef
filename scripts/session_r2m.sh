#!/bin/bash
# Round-2 late session on the K3 (redux select, early trigger, paired 4-slot ring) tree: full GPU
# suite, smoke, bench, launch list, K3 full ncu at C3, per-kernel table, primitives, probes.
set -u
mkdir -p gpurun_out
timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_m.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_m.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_m.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_m.txt
timeout 900 python bench.py > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_m.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_m.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
PROBE_VARIANTS=default timeout 600 python scripts/rerank_probe.py > gpurun_out/rerank_m.txt 2>&1; echo "rerank rc=$?"; cat gpurun_out/rerank_m.txt
PROBE_SHAPES=64:100:1024:10,128:200:1024:10,256:50:768:10,1024:50:768:10 PROBE_VARIANTS=default timeout 600 python scripts/rerank_probe.py >> gpurun_out/rerank_m.txt 2>&1; echo "rerank2 rc=$?"; tail -4 gpurun_out/rerank_m.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rerank -s 3 -c 1 -o gpurun_out/k3_c3_m python scripts/rerank_ncu.py > gpurun_out/k3_ncu_m.log 2>&1; echo "k3 ncu rc=$?"
timeout 900 ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/ktable_m.csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed python scripts/kernel_table.py > gpurun_out/ktable_m_run.log 2>&1; echo "ktable rc=$?"
python scripts/kernel_table.py --summarize gpurun_out/ktable_m.csv > gpurun_out/ktable_m.txt 2>&1; cat gpurun_out/ktable_m.txt
timeout 600 python bench_primitives.py > gpurun_out/prims_m.jsonl 2> gpurun_out/prims_m.err; echo "prims rc=$?"
timeout 1500 python bench_workflows.py > gpurun_out/workflows_m.jsonl 2>&1; echo "wf rc=$?"
timeout 600 python scripts/stream_probe.py > gpurun_out/stream_m.jsonl 2>&1; echo "stream rc=$?"
