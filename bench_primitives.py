#!/usr/bin/env python
"""Primitive-level measurements of the retrieval path at every BASELINE config.

One JSON line per config, device-timed with CUDA events (warm-up, then `--reps` launches back
to back; the corpus is larger than L2 except where noted), next to the CPU oracle (C, OpenMP,
all host threads) timed on a bounded sample of the same inputs, and the reference's modelled
latency for the batch (its hand-written profile table, "simulated").

  C1  naive RAG primitive: 16 queries x top-5 over a 10k x 384 corpus (latency-bound; also
      through a CUDA graph, `CapturedSearch`)
  C2  flat IP: 1M x 768 bf16, B=256, k=10
  C3  advanced RAG primitive: 256 questions x 4 expanded queries x top-50 over 1M x 768,
      Aggregate (200 candidates per question) -> rerank 200 -> 10 with dedup
  C4  10M x 1024, B=1024, k=100 (one GPU), and one shard at G=8 (1.25M rows)
  C5  contextual retrieval primitive: 16 queries, each top-32 over its own 48-row index
      segment (one segmented launch), then rerank 32 -> 3

    python bench_primitives.py [--configs c1,c2,c3,c4,c5] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def dev_time(fn, reps: int, warmup: int = 3) -> float:
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def cpu_search_ms(q, rows_dev, k, n_sample, threads):
    """C oracle on the first n_sample rows, scaled to the full row count (ms)."""
    import numpy as np
    import torch

    from oracle import c_oracle

    n = rows_dev.shape[0]
    m = min(n, n_sample)
    cb = rows_dev[:m].view(torch.int16).cpu().numpy().view(np.uint16)
    qb = q.bfloat16().view(torch.int16).cpu().numpy().view(np.uint16)
    c_oracle.search(qb, cb, k, nthreads=threads)  # warm
    t = time.perf_counter()
    c_oracle.search(qb, cb, k, nthreads=threads)
    return (time.perf_counter() - t) * 1000.0 * n / m, m


def roof(flops, nbytes, ms, peaks):
    tf = flops / (ms * 1e-3) / 1e12
    gbs = nbytes / (ms * 1e-3) / 1e9
    ptf, pbw = peaks["bf16_tflops"], peaks["hbm_gbs"]
    bound = "tensor" if flops / (ptf * 1e12) >= nbytes / (pbw * 1e9) else "hbm"
    return {"bound": bound, "tensor_tflops": tf, "tensor_frac": tf / ptf, "hbm_gbs": gbs,
            "hbm_frac": gbs / pbw}


def make_index(rows, dim, dev, seed=0):
    import torch

    from paper_2407_00326_b200.index import DeviceIndex

    idx = DeviceIndex(dim, rows, metric="cosine", device=dev.index)
    chunk = 1 << 20
    for a in range(0, rows, chunk):
        g = torch.Generator(device=dev).manual_seed(seed * 1000 + a // chunk)
        idx.append(torch.randn((min(chunk, rows - a), dim), generator=g, device=dev))
    torch.cuda.synchronize()
    return idx


def queries(B, dim, dev, seed=1):
    import torch

    from paper_2407_00326_b200.index import normalize_rows

    g = torch.Generator(device=dev).manual_seed(seed)
    return normalize_rows(torch.randn((B, dim), generator=g, device=dev))


def simulated(eid, load):
    from paper_2407_00326_b200 import engines as E

    prof = json.loads((ROOT / "tests" / "golden" / "ref_profiles.json").read_text())
    es = E.EngineSet.from_dict(prof["default"]["profiles"])
    return E.latency(es[eid], float(load))


def c1(args, dev, peaks, threads):
    from paper_2407_00326_b200.launcher import CapturedSearch

    N, D, B, k = 10_000, 384, 16, 5
    idx = make_index(N, D, dev)
    q = queries(B, D, dev)
    ms = dev_time(lambda: idx.search(q, k), args.reps)
    cap = CapturedSearch(idx, B, k)
    ms_graph = dev_time(lambda: cap.search(q), args.reps)
    cpu_ms, _ = cpu_search_ms(q, idx.data(), k, N, threads)
    return {"config": "C1 primitive: 10k x 384, B=16, k=5", "device_ms": ms,
            "device_ms_cuda_graph": ms_graph, "queries_per_s": B / (ms_graph * 1e-3),
            "roofline": roof(2.0 * B * N * D, N * D * 2, ms, peaks),
            "note": "corpus (7.7 MB) is L2-resident; launch-latency bound",
            "cpu_oracle_ms": cpu_ms, "cpu_threads": threads,
            "simulated_reference_ms": simulated("vdb-search0", B)}


def c2(args, dev, peaks, threads):
    N, D, B, k = 1_000_000, 768, 256, 10
    idx = make_index(N, D, dev)
    q = queries(B, D, dev)
    out = (q.new_empty((B, k), dtype=__import__("torch").float32),
           q.new_empty((B, k), dtype=__import__("torch").int32))
    ms = dev_time(lambda: idx.search(q, k, out=out), args.reps)
    cpu_ms, m = cpu_search_ms(q, idx.data(), k, 100_000, threads)
    return {"config": "C2: 1M x 768 bf16, B=256, k=10", "device_ms": ms,
            "queries_per_s": B / (ms * 1e-3),
            "roofline": roof(2.0 * B * N * D, N * D * 2, ms, peaks),
            "cpu_oracle_ms": cpu_ms, "cpu_sample_rows": m, "cpu_threads": threads,
            "simulated_reference_ms": simulated("vdb-search0", B)}


def c3(args, dev, peaks, threads):
    import torch

    N, D, Bq, E, k_s, C, k_r = 1_000_000, 768, 256, 4, 50, 200, 10
    idx = make_index(N, D, dev)
    qx = queries(Bq * E, D, dev)
    qq = queries(Bq, D, dev, seed=2)
    res = {}

    def search():
        res["s"] = idx.search(qx, k_s)

    def rerank():
        cand = res["s"][1].view(Bq, E * k_s)  # Aggregate = concatenation in slice order
        res["r"] = idx.rerank(qq, cand, k_r)

    search()
    ms_s = dev_time(search, args.reps)
    ms_r = dev_time(rerank, args.reps)
    ms_both = dev_time(lambda: (search(), rerank()), args.reps)
    from paper_2407_00326_b200.launcher import CapturedRetrieval

    chain = CapturedRetrieval(idx, Bq, E, k_s, k_r)
    ms_graph = dev_time(lambda: chain.run(qx, qq), args.reps)
    cpu_ms, m = cpu_search_ms(qx, idx.data(), k_s, 50_000, threads)
    return {"config": "C3 primitive: 256 questions x 4 queries x top-50 over 1M x 768, "
                      "Aggregate 200 -> rerank 200 -> 10 (dedup)",
            "search_ms": ms_s, "rerank_ms": ms_r, "device_ms": ms_both,
            "device_ms_cuda_graph": ms_graph,
            "questions_per_s": Bq / (ms_both * 1e-3),
            "search_roofline": roof(2.0 * Bq * E * N * D, N * D * 2, ms_s, peaks),
            "rerank_roofline": roof(2.0 * Bq * C * D, Bq * C * D * 2, ms_r, peaks),
            "cpu_oracle_search_ms": cpu_ms, "cpu_sample_rows": m, "cpu_threads": threads,
            "simulated_reference_ms": {"search": simulated("vdb-search0", Bq * E),
                                       "rerank": simulated("rerank0", C) * Bq}}


def c4(args, dev, peaks, threads):
    import torch

    out = []
    for N, label in ((10_000_000, "one GPU, whole corpus"), (1_250_000, "one shard at G=8")):
        D, B, k = 1024, 1024, 100
        idx = make_index(N, D, dev)
        q = queries(B, D, dev)
        o = (torch.empty((B, k), device=dev), torch.empty((B, k), dtype=torch.int32, device=dev))
        ms = dev_time(lambda: idx.search(q, k, out=o), max(3, args.reps // 4))
        out.append({"config": f"C4: {N} x 1024, B=1024, k=100 ({label})", "device_ms": ms,
                    "queries_per_s": B / (ms * 1e-3),
                    "roofline": roof(2.0 * B * N * D, N * D * 2, ms, peaks),
                    "simulated_reference_ms": simulated("vdb-search0", B)})
        del idx
        torch.cuda.empty_cache()
    return out


def c5(args, dev, peaks, threads):
    import torch

    nq, seg, D, k, k_r = 16, 48, 1024, 32, 3
    idx = make_index(nq * seg, D, dev)
    q = queries(nq, D, dev)
    offs = list(range(nq + 1))
    ranges = [(i * seg, (i + 1) * seg) for i in range(nq)]
    res = {}

    def search():
        res["s"] = idx.search_segmented(q, offs, ranges, k, local_ids=False)

    def rerank():
        res["r"] = idx.rerank(q, res["s"][1], k_r)

    search()
    ms_s = dev_time(search, args.reps)
    ms_r = dev_time(rerank, args.reps)
    ms_both = dev_time(lambda: (search(), rerank()), args.reps)
    from paper_2407_00326_b200.launcher import CapturedContextual

    chain = CapturedContextual(idx, offs, ranges, k, k_r, fused=False)
    ms_graph = dev_time(lambda: chain.run(q), args.reps)
    rows = torch.tensor(ranges, dtype=torch.int64, device=dev)
    ms_fused = dev_time(lambda: idx.search_rerank_segmented(q, rows, seg, k, k_r,
                                                            local_ids=False), args.reps)
    fused = CapturedContextual(idx, offs, ranges, k, k_r)
    ms_fused_graph = dev_time(lambda: fused.run(q), args.reps)
    return {"config": "C5 primitive: 16 queries, each top-32 over its own 48-row segment "
                      "(one segmented launch), rerank 32 -> 3",
            "search_ms": ms_s, "rerank_ms": ms_r, "chain_ms": ms_both,
            "chain_ms_cuda_graph": ms_graph, "fused_chain_ms": ms_fused,
            "fused_chain_ms_cuda_graph": ms_fused_graph,
            "note": "launch / latency bound (98 KB per segment)",
            "simulated_reference_ms": {"search": simulated("vdb-search0", nq),
                                       "rerank": simulated("rerank0", 32)}}


def main():
    ap = argparse.ArgumentParser(description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch

    from paper_2407_00326_b200 import _native

    _native.load()
    dev = torch.device("cuda", 0)
    p = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(p.read_text()) if p.exists() else {"bf16_tflops": 2250.0,
                                                           "hbm_gbs": 7700.0}
    threads = os.cpu_count() or 1
    for name in args.configs.split(","):
        r = globals()[name](args, dev, peaks, threads)
        for line in (r if isinstance(r, list) else [r]):
            print(json.dumps(line), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
