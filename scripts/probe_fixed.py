"""Diagnostic: fixed per-launch cost of the scan kernels (ncu --profile-from-start off).
Set TSV_DIAG=128 for setup/teardown only (single-CTA kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402

dev = torch.device("cuda", 0)
idx = DeviceIndex(384, 256, metric="ip", device=0)   # one tile: R = 1, no merge; ip: no normalize
idx.append(normalize_rows(torch.randn((256, 384), device=dev)))
q = normalize_rows(torch.randn((int(os.environ.get("PROBE_B", "16")), 384), device=dev))
for _ in range(3):
    idx.search(q, int(os.environ.get("PROBE_K", "10")))
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(3):
    idx.search(q, int(os.environ.get("PROBE_K", "10")))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
