"""Diagnostic: kernel durations of a small latency-bound search (C1: 16 queries x 10k x 384, k=5).
Run under `ncu --metrics gpu__time_duration.sum --profile-from-start off`."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402

dev = torch.device("cuda", 0)
idx = DeviceIndex(384, 10_000, metric="cosine", device=0)
idx.append(torch.randn((10_000, 384), device=dev))
q = normalize_rows(torch.randn((16, 384), device=dev))
for _ in range(5):
    idx.search(q, 5)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(3):
    idx.search(q, 5)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
