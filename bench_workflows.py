#!/usr/bin/env python
"""Workflow-level measurement of the retrieval path (BASELINE configs C1, C3, C5).

The reference's e-graphs (compiled by its optimizer: tests/golden/workflow_graphs.json) are
submitted with Poisson arrivals at the rates of pkg/configs/*.json to the mirrored
simulator, with the B200 RetrievalBackend bound at `_execute` in timing="measured" mode:
every `vdb-search0` / `rerank0` batch runs the real kernels on seeded synthetic data and the
simulator advances by the device-measured time. LLM / embedding / ingest / web primitives
stay latency-modelled exactly as in the reference.

Prints one JSON line per config: end-to-end query latency (virtual ms), and for the
retrieval engines the measured device time per batch next to the reference profile's
modelled latency for the same batch ("simulated").

    python bench_workflows.py [--configs c1_naive_10k,c3_advanced,c5_colocated] [--queries N]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
FIXTURE = ROOT / "tests" / "golden" / "workflow_graphs.json"


def poisson_arrivals(rate_qps: float, duration_s: float, seed: int, limit: int | None):
    rng = np.random.default_rng(seed)
    t, out = 0.0, []
    while True:
        t += rng.exponential(1000.0 / rate_qps)
        if t > duration_s * 1000.0 or (limit is not None and len(out) >= limit):
            return out
        out.append(t)


def restamp(raw: dict, query_id: str, app_id: str):
    from paper_2407_00326_b200.graph import parse_graph

    g = parse_graph(raw)
    g.query_id = query_id
    for node in g.nodes.values():
        node.meta.query_id = query_id
        node.meta.app_id = app_id
    return g


def pct(xs, q):
    return float(np.percentile(np.asarray(xs), q)) if xs else None


def run_config(name: str, cfg: dict, profiles: dict, limit: int | None, devices):
    import torch

    from paper_2407_00326_b200 import engines as E
    from paper_2407_00326_b200 import runtime as R
    from paper_2407_00326_b200.backend import TIMING_MEASURED, RetrievalBackend

    prof = json.loads(json.dumps(profiles))
    replicas = int(cfg.get("replicas", 1))
    for p in prof["engines"]:
        if p["engine_id"] in ("vdb-search0", "rerank0"):
            p["instances"] = replicas
    es = E.EngineSet.from_dict(prof)
    subs = []
    for ai, app in enumerate(cfg["apps"]):
        for j, t in enumerate(poisson_arrivals(app["rate_qps"], cfg["duration_s"],
                                               cfg["seed"] + ai, limit)):
            subs.append((restamp(app["graph"], f"{app['app']}-{j}", app["app"]), t, 0.0))
    subs.sort(key=lambda x: x[1])
    rows = 0
    for g, _, _ in subs:
        for node in g.nodes.values():
            if node.kind.value == "Ingestion":
                rows += max(p.items for p in node.meta.outputs.values())
    devs = [devices[i % len(devices)] for i in range(replicas)]
    backend = RetrievalBackend(dim=cfg["dim"], devices=devs,
                               arena_rows=max(1 << 16, rows * 2 + 4096), timing=TIMING_MEASURED)
    backend.warmup()
    sim, trace = R.run_queries(es, subs, R.RuntimeOptions(scheduler="topo"), backend=backend)
    torch.cuda.synchronize()
    from paper_2407_00326_b200.report import retrieval_report

    lat = [c.latency_ms for c in sim.contexts.values() if c.latency_ms is not None]
    out = {"config": name, "queries": len(subs), "completed": len(lat),
           "e2e_ms": {"mean": float(np.mean(lat)) if lat else None, "p50": pct(lat, 50),
                      "p95": pct(lat, 95)},
           "replicas": replicas, "dim": cfg["dim"], "engines": {}}
    for eid in ("vdb-search0", "rerank0"):
        bs = [b for b in trace.batches if b.engine_id == eid]
        if not bs:
            continue
        dev = [b.device_ms for b in bs]
        sim_ms = [E.latency(es[eid], b.load) for b in bs]
        out["engines"][eid] = {
            "batches": len(bs), "mean_load": float(np.mean([b.load for b in bs])),
            "device_ms": {"p50": pct(dev, 50), "p95": pct(dev, 95), "mean": float(np.mean(dev))},
            "simulated_profile_ms": {"p50": pct(sim_ms, 50), "mean": float(np.mean(sim_ms))},
        }
    out["device_report"] = retrieval_report(backend)
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--configs", default="c1_naive_10k,c3_advanced,c5_colocated")
    ap.add_argument("--queries", type=int, default=None, help="cap queries per app")
    args = ap.parse_args()
    import torch

    devices = list(range(torch.cuda.device_count()))
    data = json.loads(FIXTURE.read_text())
    for name in args.configs.split(","):
        print(json.dumps(run_config(name, data["configs"][name], data["profiles"], args.queries,
                                    devices)), flush=True)


if __name__ == "__main__":
    main()
