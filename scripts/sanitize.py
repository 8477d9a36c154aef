"""Small search / segmented search / rerank / merge / normalize calls for compute-sanitizer
(memcheck, racecheck, synccheck) on the GPU box:

    compute-sanitizer --tool memcheck python scripts/sanitize.py
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_00326_b200.index import DeviceIndex, merge_topk, normalize_rows  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    idx = DeviceIndex(256, 40_000, metric="cosine", device=0)
    idx.append(torch.randn((40_000, 256), generator=g, device=dev))
    for B, k in ((1, 5), (100, 10), (300, 10), (64, 100)):
        q = normalize_rows(torch.randn((B, 256), generator=g, device=dev))
        idx.search(q, k)
    os.environ["TSV_WIDE"] = "1"  # 256-row corpus tiles (single-CTA kernel, 96 < B <= 128)
    idx.search(normalize_rows(torch.randn((120, 256), generator=g, device=dev)), 16,
               row_range=(77, 40_000))
    del os.environ["TSV_WIDE"]
    q = normalize_rows(torch.randn((40, 256), generator=g, device=dev))
    idx.search_segmented(q, [0, 10, 25, 40], [(0, 48), (48, 3000), (3000, 40_000)], 8)
    cand = torch.randint(0, 40_000, (4, 200), generator=g, device=dev, dtype=torch.int32)
    idx.rerank(q[:4], cand, 10)
    # K3 variants: per-warp lists (default), ring + block sort, split over blocks, row offsets
    cand2 = torch.randint(0, 3000, (40, 200), generator=g, device=dev, dtype=torch.int32)
    offs = torch.arange(0, 40 * 100, 100, device=dev, dtype=torch.int32)
    idx.rerank(q, cand2, 10, row_offsets=offs)
    for knob, val in (("TSV_RERANK_SORT", "1"), ("TSV_RERANK_SPLITS", "3")):
        os.environ[knob] = val
        idx.rerank(q, cand2, 10)
        del os.environ[knob]
    # ring routing: B <= #SMs with C >= 64 -> 4 slots scored in pairs (above); more questions
    # than SMs -> 2 slots; C not a multiple of the pair stride, duplicate and invalid ids
    qb = normalize_rows(torch.randn((200, 256), generator=g, device=dev))
    cand3 = torch.randint(-1, 40_000, (200, 77), generator=g, device=dev, dtype=torch.int32)
    cand3[:, 5] = cand3[:, 4]
    idx.rerank(qb, cand3, 7)
    idx.rerank(qb[:50], cand3[:50], 7)
    s = torch.sort(torch.randn((8, 37, 16), generator=g, device=dev), dim=2, descending=True)[0]
    i = torch.arange(8 * 37 * 16, device=dev, dtype=torch.int32).reshape(8, 37, 16)
    merge_topk(s, i, 10)
    # k > 32 candidate mode: every row (<= 8192 rows), seeded (sample + candidate pass + gated
    # fallback), segmented; range-major rounds with and without lockstep (B=1024 / 2048)
    small = DeviceIndex(256, 6000, metric="cosine", device=0)
    small.append(torch.randn((6000, 256), generator=g, device=dev))
    small.search(normalize_rows(torch.randn((50, 256), generator=g, device=dev)), 100)
    big = DeviceIndex(128, 300_000, metric="cosine", device=0)
    big.append(torch.randn((300_000, 128), generator=g, device=dev))
    for B, k in ((1024, 100), (1024, 10), (2048, 10), (200, 64)):
        big.search(normalize_rows(torch.randn((B, 128), generator=g, device=dev)), k)
    idx.search_segmented(q, [0, 10, 25, 40], [(0, 48), (48, 3000), (3000, 9000)], 64)
    # one-launch searches: K2t (tcgen05, row-major) and K2s (CUDA cores, tiled); fused C5 chain
    c1 = DeviceIndex(384, 10_000, metric="cosine", device=0)
    c1.append(torch.randn((10_000, 384), generator=g, device=dev))
    c1.search(torch.randn((16, 384), generator=g, device=dev), 5)
    c1t = DeviceIndex(256, 3000, metric="ip", device=0, storage="bf16_tiled")
    c1t.append(torch.randn((3000, 256), generator=g, device=dev))
    c1t.search(torch.randn((40, 256), generator=g, device=dev), 12)
    rows = torch.tensor([[0, 48], [48, 96], [96, 103], [200, 1224]], dtype=torch.int64, device=dev)
    c1.search_rerank_segmented(torch.randn((4, 384), generator=g, device=dev), rows, 1024, 32, 3)
    f32 = DeviceIndex(64, 5000, metric="ip", device=0, storage="f32")
    f32.append(torch.randn((5000, 64), generator=g, device=dev))
    f32.search(torch.randn((20, 64), generator=g, device=dev), 10)
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
