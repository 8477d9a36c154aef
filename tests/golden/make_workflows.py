"""Compile the workflow e-graphs used by bench_workflows.py with the reference optimizer.

Run in the development container (needs /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_workflows.py
Writes workflow_graphs.json: for each BASELINE config the reference's optimized e-graph of one
query (restamped per query at bench time), the arrival process parameters from
pkg/configs/*.json, and the engine profile set.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "workflow_graphs.json"
sys.path.insert(0, str(REF / "src"))

from teola_sim import engines as E  # noqa: E402
from teola_sim import optimizer as O  # noqa: E402
from teola_sim.graph import serialize_graph  # noqa: E402
from teola_sim.workflow import QueryConfig  # noqa: E402
from teola_sim.workloads import AppKind, build_app_template  # noqa: E402

# BASELINE.json configs, mapped onto the reference apps
CONFIGS = {
    # C1: naive RAG, 10k chunks per query index, top-5; pkg/configs/colocated_rag.json "naive"
    "c1_naive_10k": {"apps": [("NAIVE_RAG_QA", {"indexing": {"chunk_count": 10000},
                                                "search": {"per_query_top_k": 5}}, 3.0)],
                     "dim": 384, "duration_s": 20.0, "seed": 1},
    # C3: advanced RAG, 4 expansions x top-50, rerank 200 -> 10; pkg/configs/advanced_rag.json
    "c3_advanced": {"apps": [("ADVANCED_RAG_QA", {
        "query_expansion": {"expansion_count": 4}, "query_embedding": {"query_count": 4},
        "search": {"query_count": 4, "per_query_top_k": 50},
        "rerank": {"candidate_count": 200, "top_k": 10}}, 2.0)],
        "dim": 1024, "duration_s": 20.0, "seed": 1},
    # C5: co-located SearchEngineGen + ContextualRetrieval, 4 qps each, 8 replicas
    "c5_colocated": {"apps": [("SEARCH_ENGINE_GEN", {}, 4.0), ("CONTEXTUAL_RETRIEVAL", {}, 4.0)],
                     "dim": 1024, "duration_s": 20.0, "seed": 1, "replicas": 8},
}


def main():
    es = E.load_profiles("default")
    out = {"profiles": es.to_dict(), "configs": {}}
    for name, cfg in CONFIGS.items():
        apps = []
        for app, params, rate in cfg["apps"]:
            kind = getattr(AppKind, app)
            g = O.compile_query(build_app_template(kind), QueryConfig(query_id="q", app_id=app,
                                                                    params=params), es)
            apps.append({"app": app, "rate_qps": rate, "graph": json.loads(serialize_graph(g))})
        out["configs"][name] = {**{k: v for k, v in cfg.items() if k != "apps"}, "apps": apps}
    OUT.write_text(json.dumps(out) + "\n")
    print(OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
