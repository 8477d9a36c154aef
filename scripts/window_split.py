"""Where a workflow batch's device window goes: bench_workflows' configs run with the library
calls bracketed by their own events and host timers. Per engine: the batch window (start event
before the library call .. end event after it, what BatchRecord.device_ms reports), the
library call's own window, and the host time of the library call."""
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench_workflows as BW  # noqa: E402
from paper_2407_00326_b200 import index as I  # noqa: E402

LOG = []


def wrap(name):
    fn = getattr(I.DeviceIndex, name)

    def inner(self, *a, **kw):
        s = kw.get("stream") or torch.cuda.current_stream(self.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        out = fn(self, *a, **kw)
        e1.record(s)
        LOG.append((name, e0, e1, (time.perf_counter() - t0) * 1e6))
        return out
    setattr(I.DeviceIndex, name, inner)


for n in ("search", "search_segmented", "rerank", "rerank_segmented", "search_rerank_segmented"):
    if hasattr(I.DeviceIndex, n):
        wrap(n)

data = json.loads(BW.FIXTURE.read_text())
for name in sys.argv[1].split(",") if len(sys.argv) > 1 else ("c1_naive_10k", "c3_advanced",
                                                               "c5_colocated"):
    LOG.clear()
    out = BW.run_config(name, data["configs"][name], data["profiles"], 20, [0])
    torch.cuda.synchronize()
    per = {}
    for n, e0, e1, h in LOG:
        per.setdefault(n, []).append((e0.elapsed_time(e1) * 1e3, h))
    med = lambda xs: round(sorted(xs)[len(xs) // 2], 1)
    print(json.dumps({"config": name,
                      "batch_window_us_p50": {k: round(v["device_ms"]["p50"] * 1e3, 1)
                                              for k, v in out["engines"].items()},
                      "library_calls": {k: {"n": len(v), "window_us_p50": med([a for a, _ in v]),
                                            "host_us_p50": med([b for _, b in v])}
                                        for k, v in per.items()}}), flush=True)
