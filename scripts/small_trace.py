"""Phase timestamps of the K2s small-scan kernel at C1's shape (TSV_SMALL_TRACE=1 prints them
from the library): 0 entry, 1 after griddepcontrol.wait, 2 queries staged, 3 rows scored,
4 block top-k written, 5 arrival counted, 6 (last block) merged."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    n, d, b, k = 10000, 384, 16, 5
    idx = DeviceIndex(d, n, metric="cosine", device=0)
    idx.append(torch.randn((n, d), generator=g, device=dev))
    q = normalize_rows(torch.randn((b, d), generator=g, device=dev))
    for _ in range(5):
        idx.search(q, k)
    torch.cuda.synchronize()
    os.environ["TSV_SMALL_TRACE"] = "1"
    for _ in range(3):
        idx.search(q, k)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
