"""Diagnostic: B=1024 search latency on a 1M x 1024 corpus in the profiler's call sequence."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402
from paper_2407_00326_b200.profiler import _time  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
idx = DeviceIndex(1024, 1_000_000, metric="cosine", device=0)
for a in range(0, 1_000_000, 1 << 18):
    idx.append(torch.randn((min(1 << 18, 1_000_000 - a), 1024), generator=g, device=dev))
for B in (1, 16, 256, 512, 1024, 1024, 512, 1024):
    q = normalize_rows(torch.randn((B, 1024), generator=g, device=dev))
    out = (torch.empty((B, 10), device=dev), torch.empty((B, 10), dtype=torch.int32, device=dev))
    ms = _time(lambda: idx.search(q, 10, out=out), reps=20)
    ms2 = _time(lambda: idx.search(q, 10, out=out), reps=20)
    print(B, round(ms, 3), round(ms2, 3), flush=True)
