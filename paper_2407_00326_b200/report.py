"""Retrieval section of the run report (SURVEY.md §5 metrics / tracing row).

Extends the reference's report (pkg/src/teola_sim/report.py:20-56, experiment.py:132-196)
with what the B200 path measured: per retrieval engine, batch count, device time
percentiles, achieved HBM GB/s and TFLOP/s from the launch records' algorithmic bytes and
flops, and their fraction of the measured peaks (MEASURED_PEAKS.json), plus a per-batch CSV.
"""

from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np

PEAKS = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def _peaks() -> dict:
    try:
        return json.loads(PEAKS.read_text())
    except (OSError, ValueError):
        return dict(FALLBACK)


def retrieval_report(backend) -> dict:
    peaks = _peaks()
    out = {}
    by_engine: dict[str, list] = {}
    for r in backend.records:
        by_engine.setdefault(r.engine_id, []).append(r)
    for eid, recs in sorted(by_engine.items()):
        ms = np.array([r.device_ms for r in recs])
        total_s = ms.sum() / 1000.0
        byt = sum(r.bytes for r in recs)
        fl = sum(r.flops for r in recs)
        gbs = byt / total_s / 1e9 if total_s > 0 else 0.0
        tfs = fl / total_s / 1e12 if total_s > 0 else 0.0
        out[eid] = {
            "batches": len(recs), "device_ms_total": float(ms.sum()),
            "device_ms_p50": float(np.percentile(ms, 50)),
            "device_ms_p95": float(np.percentile(ms, 95)),
            "achieved_gbs": gbs, "achieved_tflops": tfs,
            "frac_hbm": gbs / float(peaks.get("hbm_gbs", FALLBACK["hbm_gbs"])),
            "frac_tensor": tfs / float(peaks.get("bf16_tflops", FALLBACK["bf16_tflops"])),
        }
    return out


def write_launch_csv(backend, path) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["engine", "replica", "kind", "queries", "rows", "k", "dim", "bytes", "flops",
                    "device_ms"])
        for r in backend.records:
            w.writerow([r.engine_id, r.replica, r.kind, r.queries, r.rows, r.k, r.dim, r.bytes,
                        r.flops, f"{r.device_ms:.6f}"])
