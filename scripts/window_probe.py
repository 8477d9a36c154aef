"""Host cost of one Searching batch issued through DeviceIndex.search_segmented with the device
idle (the bench_workflows "device window" situation): host time of the call, and the CUDA-event
window from a start event recorded just before the call to an end event after it.
C1 shape: one query over its own 10k x 384 segment of a larger arena, k=5."""
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2407_00326_b200.index import DeviceIndex  # noqa: E402


def probe(dim, seg_rows, nseg, qper, k, reps=200, rotate=0, busy_ms=0.0):
    dev = torch.device("cuda:0")
    total = seg_rows * (nseg + rotate)
    idx = DeviceIndex(dim, capacity=total + 64, device=0)
    idx.append(torch.nn.functional.normalize(torch.randn(total, dim, device=dev), dim=1))
    q = torch.nn.functional.normalize(torch.randn(nseg * qper, dim, device=dev), dim=1).to(
        torch.bfloat16)
    s = torch.cuda.Stream()
    offs = [i * qper for i in range(nseg + 1)]
    ranges = [(i * seg_rows, (i + 1) * seg_rows) for i in range(nseg)]
    host, win = [], []
    for r in range(reps):
        torch.cuda.synchronize()
        if busy_ms:  # Python work between calls (a scheduler's), cooling the launch path
            junk, tb = {}, time.perf_counter()
            while (time.perf_counter() - tb) * 1e3 < busy_ms:
                for i in range(200):
                    junk[(i, len(junk))] = [i] * 8
            del junk
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        sh = (r % rotate) * seg_rows if rotate else 0
        rr = [(x + sh, y + sh) for x, y in ranges]
        a.record(s)
        idx.search_segmented(q, offs, rr, k, stream=s)
        b.record(s)
        t1 = time.perf_counter()
        b.synchronize()
        if r >= 20:
            host.append((t1 - t0) * 1e6)
            win.append(a.elapsed_time(b) * 1e3)
    # device-only: the same call back to back (device busy, host hidden)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(50):
        idx.search_segmented(q, offs, ranges, k, stream=s)
    b.record(s)
    b.synchronize()
    med = lambda xs: sorted(xs)[len(xs) // 2]
    return {"dim": dim, "seg_rows": seg_rows, "nseg": nseg, "queries_per_seg": qper, "k": k, "rotating_segments": rotate, "busy_ms": busy_ms,
            "host_us_p50": round(med(host), 1), "window_us_p50": round(med(win), 1),
            "back_to_back_us": round(a.elapsed_time(b) * 1e3 / 50, 1)}


if __name__ == "__main__":
    for cfg in ((384, 10000, 1, 1, 5), (384, 10000, 1, 16, 5), (1024, 48, 16, 1, 32),
                (1024, 2000, 4, 1, 50)):
        print(json.dumps(probe(*cfg)), flush=True)
    for cfg in ((384, 10000, 1, 1, 5), (1024, 48, 16, 1, 32)):
        print(json.dumps(probe(*cfg, rotate=40)), flush=True)
    for busy in (0.5, 2.0, 10.0):
        print(json.dumps(probe(384, 10000, 1, 1, 5, reps=80, busy_ms=busy)), flush=True)
