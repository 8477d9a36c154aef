"""K3 rerank device time at C3 / C5 shapes (diagnostic; run under gpurun).

Each variant replays a CUDA graph of 32 rerank calls whose candidate sets rotate over 8
random draws (8 x 79 MB > L2: rows come from HBM; `l2` repeats one draw), so the number is the
kernel's device time per call without the host's per-call issue cost (~15 us from Python).
Variants: ldg = register gather (TSV_RERANK_LDG=1); default = per-warp lists over cp.async rings
(ring depth / warps / splits knobs); sort = ring + block sort. PROBE_SPAN limits candidates to the first rows of the corpus."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402

VARIANTS = [("ldg", {"TSV_RERANK_LDG": "1"}), ("default", {}),
            ("lists", {"TSV_RERANK_LISTS": "1"}),
            ("lists_s3", {"TSV_RERANK_LISTS": "1", "TSV_RERANK_SLOTS": "3"}),
            ("lists_w16", {"TSV_RERANK_LISTS": "1", "TSV_RERANK_WARPS": "16"}),
            ("sort_s2", {"TSV_RERANK_SORT": "1"}),
            ("sort_bitonic", {"TSV_RERANK_SORT": "1", "TSV_RERANK_BITONIC": "1"}),
            ("sort_s3", {"TSV_RERANK_SORT": "1", "TSV_RERANK_SLOTS": "3"}),
            ("sort_s4", {"TSV_RERANK_SORT": "1", "TSV_RERANK_SLOTS": "4"}),
            ("ring_s2", {"TSV_RERANK_SLOTS": "2"}), ("ring_s3", {"TSV_RERANK_SLOTS": "3"}),
            ("ring_s4", {"TSV_RERANK_SLOTS": "4"}), ("no_net", {"TSV_RERANK_NO_NET": "1"})]
KNOBS = ("TSV_RERANK_LDG", "TSV_RERANK_SLOTS", "TSV_RERANK_WARPS", "TSV_RERANK_SPLITS",
         "TSV_RERANK_SORT", "TSV_RERANK_LISTS", "TSV_RERANK_BITONIC", "TSV_RERANK_NO_NET")


def graph_time(calls, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for fn in calls:  # warm-up grows workspaces outside the capture
            fn(s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for fn in calls:
            fn(torch.cuda.current_stream())
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / len(calls) * 1000


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    out = []
    shapes = ((1_000_000, 768, 256, 200, 10), (1_000_000, 1024, 16, 32, 3),
              (1_000_000, 1024, 256, 200, 10))
    if os.environ.get("PROBE_SHAPES"):  # "B:C:D:k,..." over a 1M-row corpus
        shapes = tuple((1_000_000, int(d), int(b), int(c), int(k)) for b, c, d, k in
                       (x.split(":") for x in os.environ["PROBE_SHAPES"].split(",")))
    variants = VARIANTS
    if os.environ.get("PROBE_VARIANTS"):
        keep = os.environ["PROBE_VARIANTS"].split(",")
        variants = [v for v in VARIANTS if v[0] in keep]
    for n, d, bq, c, k in shapes:
        idx = DeviceIndex(d, n, metric="ip", device=0)
        for a in range(0, n, 1 << 18):
            idx.append(normalize_rows(torch.randn((min(1 << 18, n - a), d), generator=g, device=dev)))
        q = normalize_rows(torch.randn((bq, d), generator=g, device=dev))
        span = int(os.environ.get("PROBE_SPAN", n))
        cands = [torch.randint(0, span, (bq, c), generator=g, device=dev, dtype=torch.int32)
                 for _ in range(8)]
        outs = [(torch.empty((bq, k), device=dev), torch.empty((bq, k), device=dev, dtype=torch.int32))
                for _ in range(32)]
        hbm = [lambda st, j=j: idx.rerank(q, cands[j % 8], k, stream=st, out=outs[j]) for j in range(32)]
        l2 = [lambda st, j=j: idx.rerank(q, cands[0], k, stream=st, out=outs[j]) for j in range(32)]
        # sequential candidates (question b gathers rows [b C, b C + C) of a rotating block):
        # the same bytes as the random gather with DRAM-friendly addresses
        seqs = [(torch.arange(bq * c, device=dev, dtype=torch.int32).view(bq, c)
                 + (r * bq * c) % max(1, n - bq * c)) for r in range(8)]
        seq = [lambda st, j=j: idx.rerank(q, seqs[j % 8], k, stream=st, out=outs[j]) for j in range(32)]
        alg = bq * c * d * 2
        for name, env in variants:
            for key in KNOBS:
                os.environ.pop(key, None)
            os.environ.update(env)
            try:
                th = graph_time(hbm)
                tl = graph_time(l2)
                ts = graph_time(seq)
            except Exception as exc:  # noqa: BLE001 - a variant that does not fit this shape
                print(f"{name} {bq}x{c}x{d}: n/a ({exc})", flush=True)
                continue
            print(f"{name} {bq}x{c}x{d}: hbm {th:6.2f} us ({alg / th / 1e3:6.0f} GB/s)  "
                  f"l2 {tl:6.2f} us  sequential-rows {ts:6.2f} us ({alg / ts / 1e3:6.0f} GB/s)",
                  flush=True)
        del idx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
