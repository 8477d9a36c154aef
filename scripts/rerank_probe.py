"""K3 rerank latency at C3 / C5 shapes (diagnostic; run under gpurun). Candidate sets rotate
over 4 random draws (4 x 79 MB > L2) for the HBM case, or repeat one draw for the L2 case.
Environment knobs select the kernel: TSV_RERANK_LDG=1 (register gather), TSV_RERANK_BUFS /
TSV_RERANK_BUF_KB (bulk-copy ring)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402


def timed(fn, reps=100):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    out = []
    for n, d, bq, c, k in ((1_000_000, 768, 256, 200, 10), (1_000_000, 1024, 16, 32, 3)):
        idx = DeviceIndex(d, n, metric="ip", device=0)
        for a in range(0, n, 1 << 18):
            idx.append(normalize_rows(torch.randn((min(1 << 18, n - a), d), generator=g, device=dev)))
        q = normalize_rows(torch.randn((bq, d), generator=g, device=dev))
        cands = [torch.randint(0, n, (bq, c), generator=g, device=dev, dtype=torch.int32)
                 for _ in range(4)]
        it = [0]

        def rot():
            it[0] = (it[0] + 1) & 3
            idx.rerank(q, cands[it[0]], k)

        out.append(f"{bq}x{c}x{d}: hbm {timed(rot):6.1f} us  l2 {timed(lambda: idx.rerank(q, cands[0], k)):6.1f} us")
        del idx
        torch.cuda.empty_cache()
    print(" | ".join(out))


if __name__ == "__main__":
    main()
