"""Real-time stream/event runtime (threaded.py replacement) and CUDA-graph capture."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as orc
from tests._util import from_dev, to_dev_bf16
from tests.test_gpu_backend import _check_outputs

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def test_stream_runtime_completes_workflows_with_real_results(cuda):
    from paper_2407_00326_b200 import engines as E
    from paper_2407_00326_b200.backend import RetrievalBackend
    from paper_2407_00326_b200.graph import parse_graph
    from paper_2407_00326_b200.launcher import run_streamed

    traces = json.loads((GOLD / "ref_traces.json").read_text())
    prof = json.loads((GOLD / "ref_profiles.json").read_text())["default"]["profiles"]
    for p_ in prof["engines"]:
        if p_["engine_id"] in ("vdb-search0", "rerank0"):
            p_["instances"] = 2  # two replicas (both on GPU 0 here; one per GPU on a node)
    es = E.EngineSet.from_dict(prof)
    graphs = []
    for name in ("advanced_c3", "contextual"):
        case = next(c for c in traces if c["case"] == name and c["scheduler"] == "topo")
        graphs += [(parse_graph(g), a) for g, a, _ in case["graphs"]]
    backend = RetrievalBackend(dim=1024, devices=[0, 0], arena_rows=1 << 16,
                               release_segments=False)
    rt, trace = run_streamed(es, graphs, backend, speed=20.0)
    assert all(ctx.finish_ms is not None for ctx in rt.contexts.values())
    gpu = [b for b in trace.batches if b.engine_id in ("vdb-search0", "rerank0")]
    assert gpu and all(b.device_ms is not None and b.device_ms > 0 for b in gpu)
    assert {b.instance_id for b in gpu} == {0, 1}
    assert _check_outputs(rt, backend) > 0
    # stream order: device consumers were dispatched before their producers finished on the
    # device, but every modelled consumer started only after the device work it depends on
    done = {}
    for t, q, n in rt.device_done:
        done[(q, n)] = max(t, done.get((q, n), 0.0))
    from paper_2407_00326_b200.graph import CONTROL_KINDS

    checked = 0
    for ctx in rt.contexts.values():
        for nid, node in ctx.graph.nodes.items():
            if rt._gpu(node) or node.kind in CONTROL_KINDS:
                continue
            for e in ctx.graph.edges:
                if e.dst == nid and (ctx.query_id, e.src) in done:
                    assert ctx.stats[nid].first_start_ms >= done[(ctx.query_id, e.src)] - 1e-6
                    checked += 1
    assert checked > 0


def test_stream_runtime_has_no_modelled_hops(cuda):
    """threaded.py:108-128 dispatches a completed node's children at once: the stream runtime
    adds no modelled Ray hop on any edge (the simulator's hop_ms + tokens * per_token_ms)."""
    from paper_2407_00326_b200 import engines as E
    from paper_2407_00326_b200.backend import RetrievalBackend
    from paper_2407_00326_b200.graph import parse_graph
    from paper_2407_00326_b200.launcher import StreamRuntime

    traces = json.loads((GOLD / "ref_traces.json").read_text())
    prof = json.loads((GOLD / "ref_profiles.json").read_text())["default"]["profiles"]
    es = E.EngineSet.from_dict(prof)
    case = next(c for c in traces if c["case"] == "advanced_c3" and c["scheduler"] == "topo")
    g = parse_graph(case["graphs"][0][0])
    rt = StreamRuntime(es, RetrievalBackend(dim=1024, arena_rows=1 << 14))
    assert all(rt._edge_delay(g, e) == 0.0 for e in g.edges)


def test_captured_search_replays_exactly(cuda):
    import torch
    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.launcher import CapturedSearch

    c = orc.make_corpus(30000, 384, seed=0)
    idx = DeviceIndex(384, 30000, device=cuda.index)
    idx.append(to_dev_bf16(c, cuda))
    cap = CapturedSearch(idx, batch=16, k=5)
    for seed in (1, 2, 3):
        q, _ = orc.make_queries(c, 16, seed=seed)
        qd = to_dev_bf16(q, cuda)
        s, i = cap.search(qd)
        es, ei = idx.search(qd, 5)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(from_dev(i), from_dev(ei))
        np.testing.assert_array_equal(from_dev(s), from_dev(es))


@pytest.mark.parametrize("metric,k_search,n", [("cosine", 50, 300_000), ("ip", 10, 40_000)])
def test_captured_retrieval_chain_replays_exactly(cuda, metric, k_search, n):
    """Search (k=50: sample pass + candidate mode; k=10: register lists) -> Aggregate -> rerank
    captured in one CUDA graph equals the same primitives called one by one, and the reranked
    lists match the oracle on the aggregated candidates."""
    import torch
    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.launcher import CapturedRetrieval

    dim, nq, e, k_r = 256, 24, 4, 10
    c = orc.make_corpus(n, dim, seed=0)
    idx = DeviceIndex(dim, n, metric=metric, device=cuda.index)
    idx.append(to_dev_bf16(c, cuda))
    cap = CapturedRetrieval(idx, nq, e, k_search, k_r)
    for seed in (1, 2):
        qx, _ = orc.make_queries(c, nq * e, seed=seed)
        qq, _ = orc.make_queries(c, nq, seed=seed + 10)
        qxd, qqd = to_dev_bf16(qx, cuda), to_dev_bf16(qq, cuda)
        rs, ri = cap.run(qxd, qqd)
        ss, si = idx.search(qxd, k_search)
        es, ei = idx.rerank(qqd, si.view(nq, e * k_search), k_r)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(from_dev(ri), from_dev(ei))
        np.testing.assert_array_equal(from_dev(rs), from_dev(es))
        if metric == "ip":  # (cosine re-normalises the stored rows)
            cand = from_dev(si).reshape(nq, e * k_search)
            exp_s, _ = orc.rerank(qq, c, cand, k_r)
            np.testing.assert_allclose(from_dev(rs), exp_s, rtol=1e-3, atol=1e-6)


def test_captured_contextual_chain_replays_exactly(cuda):
    """Segmented search (each query over its own 48-row segment, top-32, arena-row ids) ->
    rerank 32 -> 3 captured in one CUDA graph equals the primitives called one by one, for
    several query batches replayed through the same graph; an uncaptured segmented search in
    between (which reuses the rotating pinned upload slots) does not disturb the graph."""
    import torch
    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.launcher import CapturedContextual

    nq, seg, dim, k, k_r = 16, 48, 1024, 32, 3
    c = orc.make_corpus(nq * seg, dim, seed=0)
    idx = DeviceIndex(dim, nq * seg, device=cuda.index)
    idx.append(to_dev_bf16(c, cuda))
    offs = list(range(nq + 1))
    ranges = [(i * seg, (i + 1) * seg) for i in range(nq)]
    cap = CapturedContextual(idx, offs, ranges, k, k_r, fused=False)
    for seed in (1, 2, 3):
        q, _ = orc.make_queries(c, nq, seed=seed)
        qd = to_dev_bf16(q, cuda)
        idx.search_segmented(qd, [0, nq], [(0, nq * seg)], 8)  # other item lists in between
        rs, ri = cap.run(qd)
        ss, si = idx.search_segmented(qd, offs, ranges, k, local_ids=False)
        es, ei = idx.rerank(qd, si, k_r)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(from_dev(ri), from_dev(ei))
        np.testing.assert_array_equal(from_dev(rs), from_dev(es))
        gi = from_dev(ri)
        for r in range(nq):
            assert ((gi[r] >= r * seg) & (gi[r] < (r + 1) * seg)).all()


def test_captured_replay_rejects_other_shapes(cuda):
    from paper_2407_00326_b200.errors import ConfigParse
    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.launcher import CapturedSearch

    c = orc.make_corpus(5000, 128, seed=0)
    idx = DeviceIndex(128, 5000, device=cuda.index)
    idx.append(to_dev_bf16(c, cuda))
    cap = CapturedSearch(idx, batch=16, k=5)
    with pytest.raises(ConfigParse):
        cap.search(to_dev_bf16(c[:1], cuda))  # would broadcast into the 16-row buffer


def test_captured_contextual_fused_matches_oracle(cuda):
    """The default CapturedContextual (C5 at D=1024: 16 queries x own 48-row segment, top-32 ->
    rerank 3) runs ONE fused kernel per replay; results match the CPU oracle's search + rerank
    and the unfused chain within the bf16 tolerance, over several replays."""
    import torch
    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.launcher import CapturedContextual

    nq, seg, dim, k, k_r = 16, 48, 1024, 32, 3
    c = orc.make_corpus(nq * seg, dim, seed=0)
    idx = DeviceIndex(dim, nq * seg, device=cuda.index)
    idx.append(to_dev_bf16(c, cuda))
    offs = list(range(nq + 1))
    ranges = [(i * seg, (i + 1) * seg) for i in range(nq)]
    cap = CapturedContextual(idx, offs, ranges, k, k_r)
    assert cap.fused
    ref = CapturedContextual(idx, offs, ranges, k, k_r, fused=False)
    n0 = _native_launches()
    for seed in (1, 2, 3):
        q, _ = orc.make_queries(c, nq, seed=seed)
        qd = to_dev_bf16(q, cuda)
        rs, ri = cap.run(qd)
        us, ui = ref.run(qd)
        torch.cuda.synchronize()
        gs, gi = from_dev(rs), from_dev(ri)
        np.testing.assert_allclose(gs, from_dev(us), rtol=1e-3, atol=1e-6)
        for r in range(nq):
            a, e = ranges[r]
            probs = orc.check_topk(from_dev(cap.s_s)[r:r + 1], from_dev(cap.s_i)[r:r + 1],
                                   q[r:r + 1], c[a:e], k, 1e-3, id_offset=a)
            assert not probs, probs[:3]
            es, ei = orc.rerank(q[r:r + 1], c, from_dev(cap.s_i)[r:r + 1], k_r)
            np.testing.assert_allclose(gs[r:r + 1], es, rtol=1e-3, atol=1e-6)
            assert ((gi[r] >= a) & (gi[r] < e)).all()
    assert _native_launches() == n0  # replays launch no library calls from the host


def _native_launches():
    from paper_2407_00326_b200 import _native

    return _native.launch_count()


def test_stream_runtime_index_affinity(cuda):
    """Two replicas: with index-location affinity the per-query indexes stay on their home
    replica (segments pulled to the other replica only when the home one is busy), and the
    results are the same real results; without it, the least-loaded choice copies more."""
    from paper_2407_00326_b200 import engines as E
    from paper_2407_00326_b200.backend import RetrievalBackend
    from paper_2407_00326_b200.graph import parse_graph
    from paper_2407_00326_b200.launcher import StreamRuntime

    traces = json.loads((GOLD / "ref_traces.json").read_text())
    prof = json.loads((GOLD / "ref_profiles.json").read_text())["default"]["profiles"]
    for p_ in prof["engines"]:
        if p_["engine_id"] in ("vdb-search0", "rerank0"):
            p_["instances"] = 2
    copies = {}
    for affinity in (True, False):
        es = E.EngineSet.from_dict(prof)
        backend = RetrievalBackend(dim=1024, devices=[0, 0], arena_rows=1 << 16,
                                   release_segments=False)
        rt = StreamRuntime(es, backend, speed=20.0, affinity=affinity)
        for name in ("advanced_c3", "contextual"):
            case = next(c for c in traces if c["case"] == name and c["scheduler"] == "topo")
            for g, a, _ in case["graphs"]:
                rt.submit_query(parse_graph(g), a, arrival_ms=a)
        rt.run()
        assert all(ctx.finish_ms is not None for ctx in rt.contexts.values())
        assert _check_outputs(rt, backend) > 0
        copies[affinity] = sum(1 for (q, _, r) in backend.segments if r != backend.home(q))
    assert copies[True] <= copies[False]


def test_captured_objects_recycle_streams(cuda):
    """Captured searches of growing shapes created and dropped one after another on one index:
    a destroyed library stream's workspace (marked captured) must not be inherited by a new
    stream that reuses its handle (the next capture would be refused from growing it)."""
    import gc

    import torch
    from paper_2407_00326_b200.index import DeviceIndex
    from paper_2407_00326_b200.launcher import CapturedSearch

    c = orc.make_corpus(30000, 256, seed=0)
    idx = DeviceIndex(256, 30000, device=cuda.index)
    idx.append(to_dev_bf16(c, cuda))
    for b, k in ((1, 5), (16, 5), (64, 16), (200, 10), (300, 32), (1, 5), (512, 10)):
        q, _ = orc.make_queries(c, b, seed=b)
        cap = CapturedSearch(idx, b, k)
        s, i = cap.search(to_dev_bf16(q, cuda))
        torch.cuda.synchronize()
        assert not orc.check_topk(from_dev(s), from_dev(i), q, c, k, 1e-3)
        del cap
        gc.collect()
