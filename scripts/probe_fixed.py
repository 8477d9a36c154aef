"""Diagnostic: fixed per-launch cost of the scan kernels (ncu --profile-from-start off)."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402

dev = torch.device("cuda", 0)
cases = []
for n in (256, 25_600, 100_000):
    idx = DeviceIndex(384, n, metric="cosine", device=0)
    idx.append(torch.randn((n, 384), device=dev))
    for b in (16, 256):
        cases.append((idx, normalize_rows(torch.randn((b, 384), device=dev))))
for idx, q in cases:
    idx.search(q, 10)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for idx, q in cases:
    idx.search(q, 10)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
