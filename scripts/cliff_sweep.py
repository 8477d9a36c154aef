"""Shape sweep that flags performance cliffs (diagnostic; run under gpurun).

For each (rows, dim, B, k) times DeviceIndex.search (CUDA events, warm) and compares with a
plain model: max(2*B*N*D / 1.30e15, (N*D*2 + B*D*2) / 6.5e12) + 15 us. Prints one line per
shape with the measured/model ratio; ratios above ~1.5 are cliffs worth a look.
"""

from __future__ import annotations

import itertools
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows
    from paper_2407_00326_b200.profiler import _time

    _native.load()
    dev = torch.device("cuda", 0)
    shapes = []
    grid = ((100_000, 384), (1_000_000, 128), (1_000_000, 768), (3_000_000, 1024),
            (300_000, 4096))
    bks = list(itertools.product((1, 8, 64, 128, 129, 300, 512, 1000, 2048), (5, 32, 100)))
    if "--quick" in sys.argv:
        grid = ((100_000, 384), (1_000_000, 128), (1_000_000, 768))
        bks = [(1, 100), (64, 100), (129, 32), (300, 32), (256, 10), (1000, 32), (2048, 5)]
    for n, d in grid:
        for b, k in bks:
            shapes.append((n, d, b, k))
    cur = None
    idx = None
    for n, d, b, k in shapes:
        if cur != (n, d):
            idx = None
            torch.cuda.empty_cache()
            idx = DeviceIndex(d, n, metric="cosine", device=0)
            g = torch.Generator(device=dev).manual_seed(0)
            for a in range(0, n, 1 << 18):
                idx.append(torch.randn((min(1 << 18, n - a), d), generator=g, device=dev))
            cur = (n, d)
        q = normalize_rows(torch.randn((b, d), device=dev))
        ms = _time(lambda: idx.search(q, k), reps=10, min_warm_ms=30.0)
        model = max(2 * b * n * d / 1.30e15, (n * d * 2 + b * d * 2) / 6.5e12) * 1e3 + 0.015
        flag = "  <-- cliff?" if ms / model > 1.5 else ""
        print(f"N={n:>8} D={d:>4} B={b:>5} k={k:>3}  {ms:8.3f} ms  model {model:8.3f}  "
              f"ratio {ms / model:5.2f}{flag}", flush=True)


if __name__ == "__main__":
    main()
