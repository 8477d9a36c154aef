"""A/B of the k > 32 sample-pass layout in one process (diagnostic; run under gpurun): each
shape timed with the old layout (TSV_SAMPLE_MIN_TILES=1, TSV_SAMPLE_LIST32=1), 32-entry lists
only, and the default, interleaved three times."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import DeviceIndex, normalize_rows  # noqa: E402
from paper_2407_00326_b200.profiler import _time  # noqa: E402

CFG = {"old": {"TSV_SAMPLE_MIN_TILES": "1", "TSV_SAMPLE_LIST32": "1"},
       "list32": {"TSV_SAMPLE_LIST32": "1"}, "new": {}}


def main():
    dev = torch.device("cuda", 0)
    for n, d, shapes in ((1_000_000, 768, ((129, 100), (300, 100), (1024, 50))),
                         (100_000, 384, ((8, 100), (64, 100), (1024, 100))),
                         (300_000, 4096, ((129, 100), (512, 100)))):
        idx = DeviceIndex(d, n, metric="cosine", device=0)
        g = torch.Generator(device=dev).manual_seed(0)
        for a in range(0, n, 1 << 18):
            idx.append(torch.randn((min(1 << 18, n - a), d), generator=g, device=dev))
        for b, k in shapes:
            q = normalize_rows(torch.randn((b, d), device=dev))
            res = {tag: [] for tag in CFG}
            for _ in range(3):
                for tag, env in CFG.items():
                    os.environ.update(env)
                    res[tag].append(_time(lambda: idx.search(q, k), reps=10, min_warm_ms=30.0))
                    for key in env:
                        os.environ.pop(key, None)
            print(f"N={n} D={d} B={b} k={k}: " +
                  "  ".join(f"{tag} {min(v):.3f}" for tag, v in res.items()) + " ms", flush=True)
        del idx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
