"""Energy attribution of the bench step under the 1 kW power cap (diagnostic; run under gpurun).

For the bench configuration (10M x 1024 bf16, B=1024, k=10) runs the fused scan + top-k for
~3 s per variant while sampling nvidia-smi power / SM clock, and prints one JSON line per
variant with ms/step, median clock, median power and energy per step:
  base        the product path
  nofilter    TSV_DIAG=16: accumulators loaded from TMEM, no top-k filtering (wrong results)
  nostream    TSV_DIAG=32: every tile re-reads its range's first corpus tile (no HBM stream)
  both        TSV_DIAG=48
  noqload     TSV_DIAG=64: query tiles loaded for the first corpus tile only (L2->SM traffic of
              the query operand removed)
  cublas      torch.matmul(Q, C_chunk^T) over 1M-row chunks into a reused bf16 buffer (the
              same flops, score matrix written to HBM, no top-k)
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


class Sampler:
    def __init__(self):
        self.rows = []
        self.proc = subprocess.Popen(
            ["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
             "-lms", "100", "-i", "0"], stdout=subprocess.PIPE, text=True)
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            try:
                a, b = [float(x) for x in line.split(",")]
                self.rows.append((a, b))
            except ValueError:
                pass

    def stop(self):
        self.proc.terminate()
        self.proc.wait()
        self.t.join(timeout=2)
        return self.rows


def med(xs):
    xs = sorted(xs)
    return xs[len(xs) // 2] if xs else None


def run_variant(name, fn, seconds=3.0):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = Sampler()
    time.sleep(0.25)
    n0 = len(s.rows)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.time()
    steps = 0
    e0.record()
    while time.time() - t < seconds:
        for _ in range(5):
            fn()
        steps += 5
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    rows = s.stop()[n0:]
    ms = e0.elapsed_time(e1) / steps
    clk = med([r[0] for r in rows])
    pw = med([r[1] for r in rows])
    out = {"variant": name, "ms_per_step": ms, "sm_mhz": clk, "power_w": pw,
           "joules_per_step": pw * ms / 1000.0 if pw else None, "steps": steps,
           "samples": len(rows)}
    print(json.dumps(out), flush=True)
    return out


def main():
    import torch

    import bench
    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows

    _native.load()
    dev = torch.device("cuda", 0)
    N, D, B, k = 10_000_000, 1024, 1024, 10
    idx = bench.build_shard(DeviceIndex, N, D, 0, N, dev)
    q, _ = bench.make_queries(N, D, B, dev, normalize_rows)

    def search():
        idx.search(q, k)

    variants = [("base", None), ("nofilter", "16"), ("nostream", "32"), ("both", "48"),
                ("noqload", "64"), ("noqload_nostream", "96"), ("base_again", None)]
    if len(sys.argv) > 1:
        variants = [v for v in variants if v[0] in sys.argv[1:]]
    for name, diag in variants:
        if diag is None:
            os.environ.pop("TSV_DIAG", None)
        else:
            os.environ["TSV_DIAG"] = diag
        run_variant(name, search)
    os.environ.pop("TSV_DIAG", None)

    rows = idx.data()
    chunk = 1 << 20
    out = torch.empty((B, chunk), dtype=torch.bfloat16, device=dev)

    def gemm():
        for a in range(0, N, chunk):
            b = min(N, a + chunk)
            torch.matmul(q, rows[a:b].t(), out=out[:, : b - a])

    if len(sys.argv) == 1 or "cublas" in sys.argv:
        run_variant("cublas", gemm)


if __name__ == "__main__":
    main()
