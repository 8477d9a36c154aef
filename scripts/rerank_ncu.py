"""K3 at C3's shape (256 questions x 200 candidates x 768 -> 10) for one `ncu --set full`
capture per variant: three warm calls, then one call each of the default (per-warp lists) and
the ring + block-sort variant (TSV_RERANK_SORT=1), candidates drawn fresh so rows come from HBM.

    ncu --set full -k regex:rerank -s 3 -c 2 python scripts/rerank_ncu.py
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    n, d, bq, c, k = 1_000_000, int(os.environ.get("PROBE_DIM", 768)), 256, 200, 10
    idx = DeviceIndex(d, n, metric="ip", device=0)
    for a in range(0, n, 1 << 18):
        idx.append(normalize_rows(torch.randn((min(1 << 18, n - a), d), generator=g, device=dev)))
    q = normalize_rows(torch.randn((bq, d), generator=g, device=dev))
    for _ in range(3):
        idx.rerank(q, torch.randint(0, n, (bq, c), generator=g, device=dev, dtype=torch.int32), k)
    for env in ({}, {"TSV_RERANK_SORT": "1"}):
        os.environ.pop("TSV_RERANK_SORT", None)
        os.environ.update(env)
        cand = torch.randint(0, n, (bq, c), generator=g, device=dev, dtype=torch.int32)
        torch.cuda.synchronize()
        idx.rerank(q, cand, k)
        torch.cuda.synchronize()
    print("rerank ncu workload done")


if __name__ == "__main__":
    main()
