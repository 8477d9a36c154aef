"""Device latency of small, launch-bound searches (per-query-index shapes of C1 / C3 / C5)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000, (time.perf_counter() - t0) / reps * 1e6


for n, dim, b, k, metric in [(10000, 384, 1, 5, "cosine"), (10000, 384, 1, 5, "ip"),
                             (48, 1024, 1, 32, "ip"), (48, 1024, 4, 16, "ip"),
                             (10000, 384, 16, 5, "ip")]:
    idx = DeviceIndex(dim, n, metric=metric)
    idx.append(torch.randn(n, dim, device="cuda"))
    q = normalize_rows(torch.randn(b, dim, device="cuda"))
    s, i = torch.empty(b, k, device="cuda"), torch.empty(b, k, dtype=torch.int32, device="cuda")
    dev_us, wall_us = timed(lambda: idx.search(q, k, out=(s, i)))
    dev2, wall2 = timed(lambda: idx.search_segmented(q, [0, b], [(0, n)], k))
    print(f"n={n} d={dim} B={b} k={k} {metric}: search {dev_us:.1f} us dev / {wall_us:.1f} us host"
          f" | segmented {dev2:.1f} us dev / {wall2:.1f} us host")
