"""Generate the golden fixtures that pin the host-side mirror to the reference.

Run in the development container (the reference is importable only there):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
It imports the reference simulator from /root/reference/pkg/src, runs it, and writes JSON
fixtures next to this script. Nothing at test time reads /root/reference.

Fixtures:
  ref_profiles.json     the reference's bundled engine profiles (default, overlap_demo) plus
                        latency() samples and max_efficient_batch() per engine
  ref_passes.json       per app/config: the pass-1 graph, and the reference's Pass 2
                        (stage_decompose) and Pass 4 (pipeline_decode) outputs on it
  ref_traces.json       full optimized e-graphs of several apps and the reference Simulator's
                        trace events + batch records under each scheduler
  ref_batching.json     random queue snapshots and the plans form_batch_topo/_blind return
  advanced_rag_golden.json  the reference's frozen Fig-5 e-graph (tests/data)
"""

from __future__ import annotations

import json
import random
import shutil
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))

from teola_sim import engines as E  # noqa: E402
from teola_sim import optimizer as O  # noqa: E402
from teola_sim import runtime as R  # noqa: E402
from teola_sim.graph import (EGraph, MetadataProfile, PGraph, Payload, PrimitiveKind,  # noqa: E402
                             PrimitiveNode, assign_depths, serialize_graph)
from teola_sim.workflow import QueryConfig  # noqa: E402
from teola_sim.workloads import AppKind, build_app_template  # noqa: E402


def g2j(g) -> dict:
    return json.loads(serialize_graph(g))


CASES = {
    "advanced_default": (AppKind.ADVANCED_RAG_QA, {}),
    "advanced_c3": (AppKind.ADVANCED_RAG_QA, {
        "query_expansion": {"expansion_count": 4},
        "query_embedding": {"query_count": 4},
        "search": {"query_count": 4, "per_query_top_k": 50},
        "rerank": {"candidate_count": 200, "top_k": 10}}),
    "naive_256": (AppKind.NAIVE_RAG_QA, {
        "query_embedding": {"query_count": 256}, "search": {"query_count": 256}}),
    "naive_c1": (AppKind.NAIVE_RAG_QA, {
        "indexing": {"chunk_count": 640}, "query_embedding": {"query_count": 16},
        "search": {"query_count": 16, "per_query_top_k": 5}}),
    "contextual": (AppKind.CONTEXTUAL_RETRIEVAL, {}),
    "search_engine": (AppKind.SEARCH_ENGINE_GEN, {}),
}


def profiles_fixture():
    out = {}
    for name in ("default", "overlap_demo"):
        es = E.load_profiles(name)
        entry = {"profiles": es.to_dict(), "latency": {}, "b_eff": {}}
        for eid, p in es.items():
            entry["b_eff"][eid] = E.max_efficient_batch(p)
            entry["latency"][eid] = [[x, E.latency(p, x)] for x in
                                     (0, 0.5, 1, 3, 8, 16, 33, 48, 100, 200, 1000, 5000)]
        out[name] = entry
    return out


def passes_fixture():
    es = E.load_profiles("default")
    out = {}
    for name, (kind, params) in CASES.items():
        t = build_app_template(kind)
        cfg = QueryConfig(query_id="q0", app_id="a0", params=params)
        g0 = O.transform(t, cfg, es)
        g1, _ = O.prune_dependencies(g0)
        s2, f2 = O.stage_decompose(g1, es)
        p4, f4 = O.pipeline_decode(g1)
        s2p4, f24 = O.pipeline_decode(s2)
        out[name] = {"pass1": g2j(g1), "stage_decompose": [g2j(s2), f2],
                     "pipeline_decode": [g2j(p4), f4], "stage_then_pipeline": [g2j(s2p4), f24],
                     "optimized": g2j(O.optimize(g0, es, O.ALL_PASSES))}
    return out


def traces_fixture():
    es = E.load_profiles("default")
    out = []
    for name in ("advanced_default", "advanced_c3", "contextual", "search_engine", "naive_c1"):
        kind, params = CASES[name]
        t = build_app_template(kind)
        graphs = []
        for i in range(3):
            cfg = QueryConfig(query_id=f"{name}-q{i}", app_id="a0", params=params)
            graphs.append((O.optimize(O.transform(t, cfg, es), es, O.ALL_PASSES), 37.0 * i, 1.5))
        for sched in R.SCHEDULERS:
            opts = R.RuntimeOptions(scheduler=sched)
            sim, trace = R.run_queries(es, graphs, opts)
            out.append({
                "case": name, "scheduler": sched,
                "graphs": [[g2j(g), a, b] for g, a, b in graphs],
                "events": [list(e) for e in trace.events],
                "batches": [[b.engine_id, b.instance_id, b.start_ms, b.end_ms, b.load, b.cap,
                             b.phase, list(b.node_ids)] for b in trace.batches],
            })
    return out


def batching_fixture():
    rng = random.Random(2024)
    cases = []
    kinds = [PrimitiveKind.SEARCHING, PrimitiveKind.RERANKING, PrimitiveKind.EMBEDDING,
             PrimitiveKind.PREFILLING, PrimitiveKind.DECODING]
    for n in range(300):
        tasks = []
        graphs = {}
        for q in range(rng.randint(1, 5)):
            qid = f"q{q}"
            nodes = {}
            for j in range(rng.randint(1, 4)):
                kind = rng.choice(kinds[:3]) if rng.random() < 0.8 else rng.choice(kinds[3:])
                nodes[f"n{j}"] = PrimitiveNode(f"n{j}", kind, MetadataProfile(
                    outputs={"o": Payload(1, 1)}, engine_id="e", batch_items=rng.randint(1, 20),
                    token_counts={"p": rng.randint(1, 300)}, context_tokens=rng.randint(0, 200)))
            g = EGraph(nodes=nodes, edges=[], query_id=qid,
                       depth={k: rng.randint(0, 3) for k in nodes})
            graphs[qid] = g
            ctx = R.QueryContext(query_id=qid, graph=g, arrival_ms=0.0)
            for nid, node in nodes.items():
                prof = E.EngineProfile("e", "search", 1, ((1, 1),))
                task = R.NodeTask(ctx=ctx, node=node, arrival_ms=float(rng.randint(0, 30)),
                                  seq=len(tasks), loads=E.node_request_loads(node, prof))
                task.next_request = rng.randint(0, len(task.loads) - 1)
                tasks.append(task)
        rng.shuffle(tasks)
        cap = float(rng.choice([1, 3, 8, 16, 64, 500]))
        now = float(rng.randint(0, 50))
        timeout = float(rng.choice([0, 5, 10, 40]))
        desc = [{"qid": t.ctx.query_id, "node": t.node_id, "kind": t.node.kind.value,
                 "meta": t.node.meta.to_dict(), "depth": t.depth, "arrival": t.arrival_ms,
                 "seq": t.seq, "next_request": t.next_request} for t in tasks]
        index = {id(t): i for i, t in enumerate(tasks)}

        def enc(plan):
            return {"entries": [[index[id(t)], c] for t, c in plan.entries], "load": plan.load,
                    "phase": plan.phase}

        topo = R.form_batch_topo(tasks, cap, now)
        bto, wake_to = R.form_batch_blind(tasks, cap, timeout, now, bundle_mode=False)
        bpo, wake_po = R.form_batch_blind(tasks, cap, timeout, now, bundle_mode=True)
        cases.append({"tasks": desc, "cap": cap, "now": now, "timeout": timeout,
                      "topo": enc(topo), "blind_to": [enc(bto), wake_to],
                      "blind_po": [enc(bpo), wake_po]})
    return cases


def main():
    (OUT / "ref_profiles.json").write_text(json.dumps(profiles_fixture(), sort_keys=True) + "\n")
    (OUT / "ref_passes.json").write_text(json.dumps(passes_fixture(), sort_keys=True) + "\n")
    (OUT / "ref_traces.json").write_text(json.dumps(traces_fixture()) + "\n")
    (OUT / "ref_batching.json").write_text(json.dumps(batching_fixture()) + "\n")
    shutil.copyfile(REF / "tests" / "data" / "advanced_rag_golden.json",
                    OUT / "advanced_rag_golden.json")
    for p in sorted(OUT.glob("*.json")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
