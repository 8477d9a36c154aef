"""Real-time StreamRuntime at speed=1 on the reference's compiled C3 (advanced RAG) and C5
(contextual) e-graphs: for every query, the retrieval chain's wall-clock span (first retrieval
batch launched -> last retrieval batch finished on the device) against the device time of its
batches, and each batch's host assembly time (launch() call) — what VERDICT r1 item 5 / 7 ask
for. Prints one JSON line per app."""
import json
import os
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
from paper_2407_00326_b200.runtime import RuntimeOptions  # noqa: E402

GOLD = ROOT / "tests" / "golden"
REPS = 10
# PROBE_ISOLATED=1: queries arrive 50 ms apart (each chain runs alone), separating the host /
# launch path's cost from queueing behind other queries' batches
ISOLATED = os.environ.get("PROBE_ISOLATED") == "1"


def main():
    traces = json.loads((GOLD / "ref_traces.json").read_text())
    prof = json.loads((GOLD / "ref_profiles.json").read_text())["default"]["profiles"]
    if os.environ.get("PROBE_PROFILE") == "b200":
        # the retrieval engines' measured B200 profiles (profiler.py): batch limits from the
        # device, not from the reference's CPU vector store (the graphs stay the reference's)
        meas = {e["engine_id"]: e for e in json.loads(
            (ROOT / "profiles" / "b200_engines.json").read_text())["engines"]}
        prof = dict(prof, engines=[meas.get(e["engine_id"], e) for e in prof["engines"]])
    for name in ("advanced_c3", "contextual"):
        case = next(c for c in traces if c["case"] == name and c["scheduler"] == "topo")
        es = E.EngineSet.from_dict(prof)
        backend = RetrievalBackend(dim=1024, arena_rows=1 << 18, release_segments=True)
        backend.warmup()
        # time every launch() call on the host (input assembly + library calls)
        host, launches = [], []
        orig = backend.launch
        holder = {}

        def timed(profile, plan, instance, _orig=orig):
            t0 = time.perf_counter()
            t_wall = holder["rt"]._wall()
            out = _orig(profile, plan, instance)
            host.append((time.perf_counter() - t0) * 1000)
            launches.append((t_wall, profile.engine_id, {t.ctx.query_id for t, _ in plan.entries},
                             {t.node_id for t, _ in plan.entries}, out))
            return out

        backend.launch = timed
        orig_chain = backend.launch_chain

        def timed_chain(profile, plan, instance, reranks, _orig=orig_chain):
            t0 = time.perf_counter()
            t_wall = holder["rt"]._wall()
            out = _orig(profile, plan, instance, reranks)
            if out is not None:
                host.append((time.perf_counter() - t0) * 1000)
                launches.append((t_wall, profile.engine_id, {t.ctx.query_id for t, _ in plan.entries},
                                 {t.node_id for t, _ in plan.entries}, out))
            return out

        backend.launch_chain = timed_chain
        # warm-up run (first-use costs of torch / library paths), then the measured run: the
        # app's queries repeated REPS times with arrivals spread 20 ms apart
        for rep_i, reps in enumerate((1, REPS)):
            host.clear()
            launches.clear()
            rt = StreamRuntime(es, backend, speed=1.0, timeout_s=300,
                               options=RuntimeOptions(native_queue="--python-queue" not in sys.argv))
            holder["rt"] = rt
            for r in range(reps):
                for j, (g, arrival, _) in enumerate(case["graphs"]):
                    eg = parse_graph(g)
                    eg.query_id = f"{eg.query_id}-{rep_i}-{r}-{j}"
                    for node in eg.nodes.values():
                        node.meta.query_id = eg.query_id
                    if ISOLATED:  # one query in flight at a time: no queueing behind others
                        arrival = 50.0 * (r * len(case["graphs"]) + j)
                    else:
                        arrival = arrival + 20.0 * r
                    rt.submit_query(eg, arrival, arrival_ms=arrival)
            rt.run()
        torch.cuda.synchronize()
        gpu = [b for b in rt.trace.batches if b.engine_id in ("vdb-search0", "rerank0")]
        done = {}
        for t, q, n in rt.device_done:
            done.setdefault(q, []).append(t)
        # per query: the retrieval tail after its last Searching input arrived: last search
        # batch launched -> last rerank batch done on the device, against the device time of
        # the batches in that window (search stages launched before it are excluded)
        spans, dev = [], []
        for ctx in rt.contexts.values():
            q = ctx.query_id
            srch = [x for x in launches if x[1] == "vdb-search0" and q in x[2]]
            rr = [x for x in launches if x[1] == "rerank0" and q in x[2]]
            rr_nodes = {nid for nid, nd in ctx.graph.nodes.items() if nd.kind.value == "Reranking"}
            done_t = [t for t, qq, nid in rt.device_done if qq == q and nid in rr_nodes]
            if not srch or not done_t:
                continue
            t_launch = max(x[0] for x in srch)
            t_done = max(done_t)  # (a fused search -> rerank launch has no rerank batch)
            window = [x for x in srch + rr if x[0] >= t_launch]
            spans.append(t_done - t_launch)
            dev.append(sum(x[4][0].elapsed_time(x[4][1]) for x in window))
        ratio = [s / d for s, d in zip(spans, dev) if d > 0]
        print(json.dumps({
            "app": name, "isolated": ISOLATED, "profile": os.environ.get("PROBE_PROFILE", "reference"), "queries": len(rt.contexts), "gpu_batches": len(gpu),
            "chain_span_ms_p50": float(np.median(spans)), "chain_device_ms_p50": float(np.median(dev)),
            "span_over_device_p50": float(np.median(ratio)), "span_over_device_max": float(max(ratio)),
            "batch_device_ms_p50": float(np.median([b_.device_ms for b_ in gpu])),
            "host_launch_ms_p50": float(np.median(host)), "host_launch_ms_p95": float(np.percentile(host, 95)),
            "fused_chain_launches": sum(1 for r in backend.records if r.kind == "search+rerank"),
        }), flush=True)


if __name__ == "__main__":
    main()
