"""Does the scan's energy per flop depend on the corpus span it streams? (diagnostic, gpurun)

B=1024, k=10, 1024-d bf16, power-capped steady state (~2 s per variant, nvidia-smi sampled):
  full10M     one search over the 10M-row arena
  chunks8     the same 10M rows as 8 searches over 1.25M-row ranges of that arena
  shard1.25M  one search over a separate 1.25M-row arena (one C4 shard at G=8), x8 per step
Prints ms per 10M-row-equivalent step, median SM clock and power.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2407_00326_b200 import _native
    from paper_2407_00326_b200.index import DeviceIndex, normalize_rows
    from scripts.power_probe import run_variant

    _native.load()
    dev = torch.device("cuda", 0)
    N, D, B, k = 10_000_000, 1024, 1024, 10
    big = bench.build_shard(DeviceIndex, N, D, 0, N, dev)
    small = bench.build_shard(DeviceIndex, N, D, 0, N // 8, dev)
    q, _ = bench.make_queries(N, D, B, dev, normalize_rows)
    n8 = N // 8

    def full():
        big.search(q, k)

    def chunks():
        for c in range(8):
            big.search(q, k, row_range=(c * n8, (c + 1) * n8))

    def shard():
        for _ in range(8):
            small.search(q, k)

    for name, fn in (("full10M", full), ("chunks8", chunks), ("shard1.25M", shard),
                     ("full10M_again", full)):
        run_variant(name, fn, seconds=2.0)


if __name__ == "__main__":
    main()
