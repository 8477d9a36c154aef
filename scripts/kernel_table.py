"""Every kernel of the retrieval path once, at a representative size, for a per-kernel ncu table
(diagnostic; run under gpurun):

  ncu --profile-from-start off --clock-control none --csv --log-file gpurun_out/ktable.csv \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed python scripts/kernel_table.py
  python scripts/kernel_table.py --summarize gpurun_out/ktable.csv

A warm-up pass runs everything first; only the second pass is inside the profiler range.
"""

from __future__ import annotations

import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CASES = [
    ("K5 normalize", "ingest 1M x 1024 fp32 rows -> L2-normalised bf16"),
    ("K1 pair k=10", "10M x 1024, B=1024, k=10 (bench config)"),
    ("K4 range merge", "74..296 ranges x 10 -> 10, B=1024"),
    ("K1 sample + K4 + seed floor", "k=100 seeding pass (1/32 of every range)"),
    ("K1c candidate", "10M x 1024, B=1024, k=100 main pass"),
    ("cand select", "B=1024 candidate rows -> top 100"),
    ("K1 single-CTA B=16", "10M x 1024, B=16, k=10 (HBM-bound)"),
    ("K2 segmented", "16 queries x own 48-row segment, k=32 (C5)"),
    ("K3 rerank", "256 questions x 200 candidates x 768 -> 10 (C3)"),
    ("K1f fp32 mode", "1M x 1024 fp32 (3xTF32), B=1024, k=10"),
    ("K2t one-launch search", "10k x 384, B=16, k=5 (C1; tcgen05, rows on M)"),
    ("K2s one-launch search", "10k x 384, B=16, k=5 (C1; CUDA-core path, TSV_NO_TINY)"),
    ("K3s fused contextual chain", "16 queries x own 48-row segment, top-32 -> rerank 3 (C5)"),
]
# (K6, the peer exchange, is not in this table: ncu serialises kernels, so rank 0's exchange waits
# for a rank whose kernel cannot start until it finishes, and ends at its timeout. Its latency
# with every rank in flight comes from scripts/k6_probe.py.)


def run():
    import torch

    import bench
    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows

    _native.load()
    dev = torch.device("cuda", 0)
    N, D = 10_000_000, 1024
    idx = bench.build_shard(DeviceIndex, N, D, 0, N, dev)
    q1024, _ = bench.make_queries(N, D, 1024, dev, normalize_rows)
    q16 = q1024[:16].contiguous()
    raw = torch.randn((1 << 20, D), device=dev)
    seg_idx = DeviceIndex(D, 16 * 48, device=0)
    seg_idx.append(normalize_rows(torch.randn((16 * 48, D), device=dev)))
    c3 = DeviceIndex(768, 1 << 20, device=0)
    c3.append(normalize_rows(torch.randn((1 << 20, 768), device=dev)))
    q3 = normalize_rows(torch.randn((256, 768), device=dev))
    cand = torch.randint(0, 1 << 20, (256, 200), dtype=torch.int32, device=dev)
    seg_q = normalize_rows(torch.randn((16, D), device=dev))
    f32 = DeviceIndex(D, 1 << 20, metric="cosine", device=0, storage="f32")
    f32.append(torch.randn((1 << 20, D), device=dev))
    qf = torch.randn((1024, D), device=dev)
    c1 = DeviceIndex(384, 10_000, metric="cosine", device=0)
    c1.append(torch.randn((10_000, 384), device=dev))
    qc1 = torch.randn((16, 384), device=dev)
    seg_rows = torch.tensor([[48 * s, 48 * s + 48] for s in range(16)], dtype=torch.int64,
                            device=dev)
    import os

    def one_pass():
        normalize_rows(raw)
        idx.search(q1024, 10)
        idx.search(q1024, 100)
        idx.search(q16, 10)
        seg_idx.search_segmented(seg_q, list(range(17)), [(48 * s, 48 * s + 48) for s in range(16)],
                                 32)
        c3.rerank(q3, cand, 10)
        f32.search(qf, 10)
        c1.search(qc1, 5)
        os.environ["TSV_NO_TINY"] = "1"
        c1.search(qc1, 5)
        del os.environ["TSV_NO_TINY"]
        seg_idx.search_rerank_segmented(seg_q, seg_rows, 48, 32, 3, local_ids=False)
        torch.cuda.synchronize()

    one_pass()
    torch.cuda.profiler.start()
    one_pass()
    torch.cuda.profiler.stop()
    print("kernel_table pass done")


def summarize(path, peaks_path=ROOT / "MEASURED_PEAKS.json"):
    peaks = json.loads(Path(peaks_path).read_text()) if Path(peaks_path).exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    launches: dict = {}
    order = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"])
        if key not in launches:
            launches[key] = {}
            order.append(key)
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3,
                 "nsecond": 1e-9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                 "%": 1}.get(unit, 1)
        launches[key][d["Metric Name"]] = v * scale
    print(f"{'kernel':58s} {'time':>10s} {'DRAM rd+wr':>11s} {'GB/s':>8s} {'of HBM':>7s} "
          f"{'tensor':>7s}")
    for key in order:
        m = launches[key]
        t = m.get("gpu__time_duration.sum", 0.0)
        by = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        gbs = by / t / 1e9 if t else 0.0
        ten = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        name = key[1][:58]
        print(f"{name:58s} {t * 1e6:9.1f}us {by / 1e6:9.1f}MB {gbs:8.0f} {gbs / hbm:7.2f} "
              f"{ten:6.1f}%")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        run()
