"""Host cost of the pieces of one small search call (C1: one query over a 10k x 384 segment,
k=5), warm (back-to-back) and cold (after `busy_ms` of unrelated Python work, as inside a
scheduler loop): a trivial ctypes call into libtsv, two torch.empty outputs, the C-ABI search
with preallocated outputs, and the full DeviceIndex.search_segmented wrapper."""
import ctypes
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2407_00326_b200 import _native as nat  # noqa: E402
from paper_2407_00326_b200.index import DeviceIndex, _stream_handle  # noqa: E402


def busy(ms):
    junk, tb = {}, time.perf_counter()
    while (time.perf_counter() - tb) * 1e3 < ms:
        for i in range(200):
            junk[(i, len(junk))] = [i] * 8


def main():
    dev = torch.device("cuda:0")
    idx = DeviceIndex(384, capacity=10064, device=0)
    idx.append(torch.nn.functional.normalize(torch.randn(10000, 384, device=dev), dim=1))
    q = torch.nn.functional.normalize(torch.randn(1, 384, device=dev), dim=1).to(torch.bfloat16)
    s = torch.cuda.Stream()
    lib = nat.load()
    out_s = torch.empty((1, 5), dtype=torch.float32, device=dev)
    out_i = torch.empty((1, 5), dtype=torch.int32, device=dev)
    sh = _stream_handle(s, idx.device)
    qo = (ctypes.c_int32 * 2)(0, 1)
    rb = (ctypes.c_int64 * 1)(0)
    re = (ctypes.c_int64 * 1)(10000)

    pieces = {
        "ctypes_trivial": lambda: lib.tsv_abi_version(),
        "torch_empty_x2": lambda: (torch.empty((1, 5), dtype=torch.float32, device=dev),
                                   torch.empty((1, 5), dtype=torch.int32, device=dev)),
        "event_record": lambda: torch.cuda.Event().record(s),
        "capi_search": lambda: lib.tsv_search(idx._h, q.data_ptr(), 0, 1, 5, 0, 10000, 0,
                                              out_s.data_ptr(), out_i.data_ptr(), sh),
        "capi_search_segmented": lambda: lib.tsv_search_segmented(
            idx._h, q.data_ptr(), 0, 1, ctypes.cast(qo, ctypes.c_void_p),
            ctypes.cast(rb, ctypes.c_void_p), ctypes.cast(re, ctypes.c_void_p), 5, 1,
            out_s.data_ptr(), out_i.data_ptr(), sh),
        "wrapper_search_segmented": lambda: idx.search_segmented(q, [0, 1], [(0, 10000)], 5,
                                                                 stream=s),
    }
    for busy_ms in (0.0, 10.0):
        row = {"busy_ms": busy_ms}
        for name, fn in pieces.items():
            ts = []
            for r in range(60):
                torch.cuda.synchronize()
                if busy_ms:
                    busy(busy_ms)
                t0 = time.perf_counter()
                fn()
                ts.append((time.perf_counter() - t0) * 1e6)
            ts = sorted(ts[10:])
            row[name] = round(ts[len(ts) // 2], 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
