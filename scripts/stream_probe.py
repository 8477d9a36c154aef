"""Real-time StreamRuntime at speed=1 on the reference's compiled C3 (advanced RAG) and C5
(contextual) e-graphs: for every query, the retrieval chain's wall-clock span (first retrieval
batch launched -> last retrieval batch finished on the device) against the device time of its
batches, and each batch's host assembly time (launch() call) — what VERDICT r1 item 5 / 7 ask
for. Prints one JSON line per app."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2407_00326_b200 import engines as E  # noqa: E402
from paper_2407_00326_b200.backend import RetrievalBackend  # noqa: E402
from paper_2407_00326_b200.graph import parse_graph  # noqa: E402
from paper_2407_00326_b200.launcher import StreamRuntime  # noqa: E402

GOLD = ROOT / "tests" / "golden"


def main():
    traces = json.loads((GOLD / "ref_traces.json").read_text())
    prof = json.loads((GOLD / "ref_profiles.json").read_text())["default"]["profiles"]
    for name in ("advanced_c3", "contextual"):
        case = next(c for c in traces if c["case"] == name and c["scheduler"] == "topo")
        es = E.EngineSet.from_dict(prof)
        backend = RetrievalBackend(dim=1024, arena_rows=1 << 16, release_segments=False)
        backend.warmup()
        # time every launch() call on the host (input assembly + library calls)
        host = []
        orig = backend.launch

        def timed(profile, plan, instance, _orig=orig):
            t0 = time.perf_counter()
            out = _orig(profile, plan, instance)
            host.append((time.perf_counter() - t0) * 1000)
            return out

        backend.launch = timed
        rt = StreamRuntime(es, backend, speed=1.0, timeout_s=120)
        for g, arrival, _ in case["graphs"]:
            rt.submit_query(parse_graph(g), arrival, arrival_ms=arrival)
        rt.run()
        torch.cuda.synchronize()
        gpu = [b for b in rt.trace.batches if b.engine_id in ("vdb-search0", "rerank0")]
        done = {}
        for t, q, n in rt.device_done:
            done.setdefault(q, []).append(t)
        spans, dev = [], []
        for q in {b_.node_ids[0].split("/")[0] for b_ in gpu} | set(done):
            pass
        by_q = {}
        for b_ in gpu:
            for nid in b_.node_ids:
                by_q.setdefault(nid.split("::")[0], []).append(b_)
        # batches carry node ids; map them to queries through the runtime's contexts
        q_of = {}
        for ctx in rt.contexts.values():
            for nid in ctx.graph.nodes:
                q_of[(ctx.query_id, nid)] = ctx.query_id
        per_q = {}
        for b_ in gpu:
            qs = {ctx.query_id for ctx in rt.contexts.values()
                  for nid in b_.node_ids if nid in ctx.graph.nodes}
            for q in qs:
                per_q.setdefault(q, []).append(b_)
        for q, bs in per_q.items():
            first = min(b_.start_ms for b_ in bs)
            last = max(done.get(q, [max(b_.end_ms for b_ in bs)]))
            spans.append(last - first)
            dev.append(sum(b_.device_ms for b_ in bs))
        ratio = [s / d for s, d in zip(spans, dev) if d > 0]
        print(json.dumps({
            "app": name, "queries": len(rt.contexts), "gpu_batches": len(gpu),
            "chain_span_ms_p50": float(np.median(spans)), "chain_device_ms_p50": float(np.median(dev)),
            "span_over_device_p50": float(np.median(ratio)), "span_over_device_max": float(max(ratio)),
            "batch_device_ms_p50": float(np.median([b_.device_ms for b_ in gpu])),
            "host_launch_ms_p50": float(np.median(host)), "host_launch_ms_p95": float(np.percentile(host, 95)),
        }), flush=True)


if __name__ == "__main__":
    main()
