"""Where does the e2e loop lose time against the device-resident loop? (diagnostic, gpurun)

Bench configuration (10M x 1024, B=1024, k=10). Alternates blocks of 5 steps of several loop
variants (same clocks for all) and prints ms/step per variant:
  dev      search(q_dev) back to back
  events   + the e2e loop's cross-stream event waits, no copies
  h2d      + the pinned host->device query upload on the copy stream
  d2h      + the device->host result download on the copy stream
  e2e      both copies (bench.py's e2e loop)
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

    _native.load()
    dev = torch.device("cuda", 0)
    N, D, B, k = 10_000_000, 1024, 1024, 10
    idx = bench.build_shard(DeviceIndex, N, D, 0, N, dev)
    q_dev, _ = bench.make_queries(N, D, B, dev, normalize_rows)
    q_host = torch.empty((B, D), dtype=torch.bfloat16, pin_memory=True)
    q_host.copy_(q_dev)
    s_out = [torch.empty((B, k), dtype=torch.float32, device=dev) for _ in range(2)]
    i_out = [torch.empty((B, k), dtype=torch.int32, device=dev) for _ in range(2)]
    h_s = [torch.empty((B, k), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    h_i = [torch.empty((B, k), dtype=torch.int32, pin_memory=True) for _ in range(2)]
    q_bufs = [torch.empty_like(q_dev), torch.empty_like(q_dev)]
    copy = torch.cuda.Stream(dev)
    comp = torch.cuda.current_stream(dev)

    def loop(steps, h2d, d2h, events):
        up = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [torch.cuda.Event(), torch.cuda.Event()]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        if not events:
            for st in range(steps):
                idx.search(q_dev, k, out=(s_out[st & 1], i_out[st & 1]))
        else:
            copy.wait_stream(comp)
            with torch.cuda.stream(copy):
                if h2d:
                    q_bufs[0].copy_(q_host, non_blocking=True)
                up[0].record(copy)
            for st in range(steps):
                b = st & 1
                if st + 1 < steps:
                    nb = b ^ 1
                    with torch.cuda.stream(copy):
                        if st >= 1:
                            copy.wait_event(freed[nb])
                        if h2d:
                            q_bufs[nb].copy_(q_host, non_blocking=True)
                        up[nb].record(copy)
                comp.wait_event(up[b])
                idx.search(q_bufs[b] if h2d else q_dev, k, out=(s_out[b], i_out[b]))
                freed[b].record(comp)
                done[b].record(comp)
                with torch.cuda.stream(copy):
                    copy.wait_event(done[b])
                    if d2h:
                        h_s[b].copy_(s_out[b], non_blocking=True)
                        h_i[b].copy_(i_out[b], non_blocking=True)
            comp.wait_stream(copy)
        e1.record(comp)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    variants = {"dev": (False, False, False), "events": (False, False, True),
                "h2d": (True, False, True), "d2h": (False, True, True), "e2e": (True, True, True)}
    for _ in range(5):
        idx.search(q_dev, k)
    tot = {n: 0.0 for n in variants}
    steps = 0
    for rep in range(6):
        for n, (a, b, c) in variants.items():
            tot[n] += loop(5, a, b, c)
        steps += 5
    print(json.dumps({n: round(v / steps, 3) for n, v in tot.items()}), flush=True)


if __name__ == "__main__":
    main()
