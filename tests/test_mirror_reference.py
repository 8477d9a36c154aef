"""The host-side mirror reproduces the reference exactly (fixtures from tests/golden/make_golden.py).

Pins: latency tables and B_eff (engines.py:85-140), Pass 2 / Pass 4 stage splitting and
Aggregate insertion (optimizer.py:536-878), batch formation (runtime.py:189-339) and whole
simulated traces (runtime.py:350-656) — the structure the GPU path plugs into."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from paper_2407_00326_b200 import engines as E
from paper_2407_00326_b200 import runtime as R
from paper_2407_00326_b200 import stages as S
from paper_2407_00326_b200.sched import TopoQueue
from paper_2407_00326_b200.graph import (EGraph, MetadataProfile, PrimitiveKind, PrimitiveNode,
                                         parse_graph, serialize_graph)

GOLD = Path(__file__).resolve().parent / "golden"


def load(name):
    return json.loads((GOLD / name).read_text())


@pytest.fixture(scope="module")
def profiles():
    return load("ref_profiles.json")


def test_latency_and_beff_match_reference(profiles):
    for name, entry in profiles.items():
        es = E.EngineSet.from_dict(entry["profiles"])
        for eid, samples in entry["latency"].items():
            for load, ms in samples:
                assert E.latency(es[eid], load) == pytest.approx(ms, abs=1e-12), (name, eid, load)
        for eid, beff in entry["b_eff"].items():
            assert E.max_efficient_batch(es[eid]) == beff, (name, eid)
    # the values SURVEY.md §8a a5 quotes
    d = E.EngineSet.from_dict(profiles["default"]["profiles"])
    assert d.b_eff("vdb-search0") == 16 and d.b_eff("rerank0") == 64


PASS_CASES = list(load("ref_passes.json").items())


@pytest.mark.parametrize("name,case", PASS_CASES, ids=[c[0] for c in PASS_CASES])
def test_stage_passes_match_reference(name, case, profiles):
    es = E.EngineSet.from_dict(profiles["default"]["profiles"])
    g1 = parse_graph(case["pass1"])
    ref_s2, ref_f2 = case["stage_decompose"]
    s2, f2 = S.stage_decompose(g1, es)
    assert f2 == ref_f2
    assert json.loads(serialize_graph(s2)) == ref_s2
    ref_p4, ref_f4 = case["pipeline_decode"]
    p4, f4 = S.pipeline_decode(g1)
    assert f4 == ref_f4
    assert json.loads(serialize_graph(p4)) == ref_p4
    ref_sp, ref_fsp = case["stage_then_pipeline"]
    sp, fsp = S.pipeline_decode(s2)
    assert fsp == ref_fsp and json.loads(serialize_graph(sp)) == ref_sp


def test_golden_search_aggregate_rerank_fragment():
    """Fig-5 golden (pkg/tests/data/advanced_rag_golden.json): 3 Searching stages of 1 query x
    top-16 with slices (16i, 16i+16, 48) -> Aggregate(48) -> Reranking(48 -> 3)."""
    g = parse_graph((GOLD / "advanced_rag_golden.json").read_text())
    rerank = g.nodes["rerank.rerank"]
    assert rerank.kind is PrimitiveKind.RERANKING and rerank.meta.batch_items == 48
    feeds = [e.src for e in g.edges if e.dst == "rerank.rerank" and e.key == "candidate_chunks"]
    assert len(feeds) == 1 and g.nodes[feeds[0]].kind is PrimitiveKind.AGGREGATE
    agg = feeds[0]
    assert g.nodes[agg].meta.outputs["candidate_chunks"].items == 48
    stages = sorted(e.src for e in g.edges if e.dst == agg)
    assert len(stages) == 3
    for i, sid in enumerate(stages):
        n = g.nodes[sid]
        assert n.kind is PrimitiveKind.SEARCHING and n.meta.batch_items == 1
        assert n.meta.slice_of["candidate_chunks"] == (16 * i, 16 * i + 16, 48)
        assert S.stage_query_range(n, "candidate_chunks") == (i, i + 1)
    # canonical round trip through the mirror's IR is byte-identical
    assert serialize_graph(g) == serialize_graph(parse_graph(serialize_graph(g)))


def test_optimized_advanced_graph_isomorphic_to_golden():
    opt = parse_graph(load("ref_passes.json")["advanced_default"]["optimized"])
    gold = parse_graph((GOLD / "advanced_rag_golden.json").read_text())
    assert sorted(n.shape_label() for n in opt.nodes.values()) == sorted(
        n.shape_label() for n in gold.nodes.values())
    assert len(opt.edges) == len(gold.edges)


TRACE_CASES = load("ref_traces.json")


@pytest.mark.parametrize("native", [True, False], ids=["native-queue", "python-queue"])
@pytest.mark.parametrize("case", TRACE_CASES, ids=[f"{c['case']}-{c['scheduler']}" for c in TRACE_CASES])
def test_simulated_trace_matches_reference(case, native, profiles):
    if not native and case["scheduler"] != "topo":
        pytest.skip("the native queue serves the topo scheduler only")
    es = E.EngineSet.from_dict(profiles["default"]["profiles"])
    subs = [(parse_graph(g), a, b) for g, a, b in case["graphs"]]
    sim, trace = R.run_queries(es, subs, R.RuntimeOptions(scheduler=case["scheduler"],
                                                          native_queue=native))
    assert [list(e) for e in trace.events] == case["events"]
    got = [[b.engine_id, b.instance_id, b.start_ms, b.end_ms, b.load, b.cap, b.phase,
            list(b.node_ids)] for b in trace.batches]
    assert got == case["batches"]


def _tasks(desc):
    graphs: dict[str, EGraph] = {}
    ctxs = {}
    tasks = []
    for d in desc:
        g = graphs.setdefault(d["qid"], EGraph(query_id=d["qid"]))
        node = PrimitiveNode(d["node"], PrimitiveKind(d["kind"]), MetadataProfile.from_dict(d["meta"]))
        g.nodes[d["node"]] = node
        g.depth[d["node"]] = d["depth"]
        ctx = ctxs.setdefault(d["qid"], R.QueryContext(query_id=d["qid"], graph=g, arrival_ms=0.0))
        prof = E.EngineProfile("e", "search", 1, ((1, 1),))
        t = R.NodeTask(ctx=ctx, node=node, arrival_ms=d["arrival"], seq=d["seq"],
                       loads=E.node_request_loads(node, prof))
        t.next_request = d["next_request"]
        tasks.append(t)
    return tasks


def test_batch_formation_matches_reference():
    cases = load("ref_batching.json")
    for c in cases:
        tasks = _tasks(c["tasks"])
        idx = {id(t): i for i, t in enumerate(tasks)}

        def enc(plan):
            return {"entries": [[idx[id(t)], n] for t, n in plan.entries], "load": plan.load,
                    "phase": plan.phase}

        assert enc(R.form_batch_topo(tasks, c["cap"], c["now"])) == c["topo"]
        # the native engine queue (csrc/tsv_sched.cpp) forms the same batch
        nq = TopoQueue(R.EPS)
        for t in tasks:
            nq.push(t)
        assert enc(nq.form(c["cap"])) == c["topo"]
        nq.close()
        p, w = R.form_batch_blind(tasks, c["cap"], c["timeout"], c["now"], bundle_mode=False)
        assert [enc(p), w] == c["blind_to"]
        p, w = R.form_batch_blind(tasks, c["cap"], c["timeout"], c["now"], bundle_mode=True)
        assert [enc(p), w] == c["blind_po"]


# ---- behaviour tests mirrored from the reference's own suite -------------
def test_select_instance_rules():
    a, b = E.EngineInstance(0), E.EngineInstance(1)
    a.executed_requests, b.executed_requests = 5, 3
    assert E.select_instance([a, b], "search", 0.0) is b
    a.kv_occupied = b.kv_occupied = 100
    assert E.select_instance([a, b], "llm", 0.0) is a
    c, d = E.EngineInstance(0, busy_until=50.0), E.EngineInstance(1)
    assert E.select_instance([c, d], "search", 10.0) is d
    assert E.select_instance([c], "search", 10.0) is None


def test_max_efficient_batch_rules():
    def prof(table, slots=16):
        return E.EngineProfile("e", "embedding", 1, tuple(table), max_slots=slots)
    assert E.max_efficient_batch(prof([(4, 150), (16, 450)])) == 16
    assert E.max_efficient_batch(prof([(1, 100), (64, 100)], 64)) == 64
    assert E.max_efficient_batch(prof([(4, 40), (16, 160)], 64)) == 4


def test_empty_batch_rejected(profiles):
    from paper_2407_00326_b200.errors import CapacityExceeded

    es = E.EngineSet.from_dict(profiles["default"]["profiles"])
    sim = R.Simulator(es)
    with pytest.raises(CapacityExceeded):
        sim._execute(es["vdb-search0"], R.BatchPlan(), 0.0)


def test_searching_cardinality_and_split():
    """Searching: batch_items = query_count, outputs = query_count x per_query_top_k
    (optimizer.py:178-197); 40 queries at B_eff 16 -> stages of 16/16/8 queries."""
    from paper_2407_00326_b200.graph import Edge, PGraph, to_egraph

    node = S.searching_node("search", "vdb-search0", {"query_count": 40, "per_query_top_k": 10},
                            ("index", "query_vectors"), "top")
    assert node.meta.batch_items == 40 and node.meta.outputs["top"].items == 400
    g = PGraph(nodes={node.node_id: node}, edges=[], query_id="q")
    es = E.EngineSet.from_profiles([E.EngineProfile("vdb-search0", "search", 1, ((1, 8), (8, 20)))])
    out, fired = S.stage_decompose(g, es)
    assert fired
    spans = sorted(S.stage_query_range(n, "top") for n in out.nodes.values())
    assert spans == [(0, 16), (16, 32), (32, 40)]
    assert sum(n.meta.outputs["top"].items for n in out.nodes.values()) == 400
    assert to_egraph(out).depth


def test_requests_span_batches_and_slot_discipline(profiles):
    es = E.EngineSet.from_dict(profiles["default"]["profiles"])
    from paper_2407_00326_b200.graph import PGraph, to_egraph

    node = S.searching_node("search", "vdb-search0", {"query_count": 40, "per_query_top_k": 3},
                            (), "top")
    g = to_egraph(PGraph(nodes={node.node_id: node}, edges=[], query_id="q0"))
    sim, trace = R.run_queries(es, [(g, 0.0, 0.0)])
    loads = [b.load for b in trace.batches]
    assert loads == [16.0, 16.0, 8.0]
    assert all(b.load <= b.cap for b in trace.batches)


def test_determinism_identical_traces(profiles):
    es = E.EngineSet.from_dict(profiles["default"]["profiles"])
    case = TRACE_CASES[0]
    runs = []
    for _ in range(2):
        subs = [(parse_graph(g), a, b) for g, a, b in case["graphs"]]
        runs.append(R.run_queries(es, subs)[1].rows())
    assert runs[0] == runs[1]


def test_b200_measured_profiles_change_the_split(profiles):
    """With the reference profile a 1024-query Searching node splits into 64 stages of 16
    (B_eff 16); with the B200-measured profile (profiles/b200_engines.json,
    written by paper_2407_00326_b200/profiler.py on a B200) it stays one launch."""
    from pathlib import Path

    from paper_2407_00326_b200.graph import PGraph

    ref = E.EngineSet.from_dict(profiles["default"]["profiles"])
    b200 = E.EngineSet.from_dict(json.loads(
        (Path(__file__).resolve().parents[1] / "profiles" / "b200_engines.json").read_text()))
    node = S.searching_node("search", "vdb-search0", {"query_count": 1024, "per_query_top_k": 10},
                            (), "top")
    g = PGraph(nodes={node.node_id: node}, edges=[], query_id="q")
    out_ref, _ = S.stage_decompose(g, ref)
    out_b200, fired = S.stage_decompose(g, b200)
    assert len(out_ref.nodes) == 64
    assert E.max_efficient_batch(b200["vdb-search0"]) >= 256
    assert len(out_b200.nodes) == 1024 // int(E.max_efficient_batch(b200["vdb-search0"]))
