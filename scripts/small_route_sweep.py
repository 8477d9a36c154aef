"""Routing check for the one-launch searches (K2t / K2s): for small shapes around the routing
limits, the device time per search as a CUDA-graph replay with the default routing vs the
general scan (TSV_NO_SMALL=1) and vs K2s (TSV_NO_TINY=1). One line per shape; 'slower' marks
shapes where the default route loses to the general scan by more than 5%."""
import itertools
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_00326_b200.index import DeviceIndex  # noqa: E402
from paper_2407_00326_b200.launcher import CapturedSearch  # noqa: E402


def replay_us(idx, q, k, env, reps=50):
    for key in ("TSV_NO_SMALL", "TSV_NO_TINY"):
        os.environ.pop(key, None)
    os.environ.update(env)
    cap = CapturedSearch(idx, q.shape[0], k)
    cap.search(q)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        cap.graph.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    worse = 0
    for d in (384, 1024):
        for n in (2_000, 10_000, 30_000, 65_000):
            idx = DeviceIndex(d, n, metric="cosine", device=0)
            idx.append(torch.randn((n, d), generator=g, device=dev))
            for b, k in itertools.product((1, 16, 64), (5, 16)):
                q = torch.randn((b, d), generator=g, device=dev)
                t_def = replay_us(idx, q, k, {})
                t_gen = replay_us(idx, q, k, {"TSV_NO_SMALL": "1"})
                t_k2s = replay_us(idx, q, k, {"TSV_NO_TINY": "1"})
                flag = "slower" if t_def > 1.05 * t_gen else ""
                worse += bool(flag)
                print(f"D={d} N={n} B={b} k={k}: default {t_def:7.1f} us  general {t_gen:7.1f} us  "
                      f"K2s-route {t_k2s:7.1f} us {flag}", flush=True)
            del idx
    for key in ("TSV_NO_SMALL", "TSV_NO_TINY"):
        os.environ.pop(key, None)
    print("shapes where the default route is >5% slower than the general scan:", worse)


if __name__ == "__main__":
    main()
