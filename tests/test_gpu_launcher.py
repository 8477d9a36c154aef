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
    backend = RetrievalBackend(dim=256, devices=[0, 0], arena_rows=1 << 16)
    rt, trace = run_streamed(es, graphs, backend, speed=20.0)
    assert all(ctx.finish_ms is not None for ctx in rt.contexts.values())
    gpu = [b for b in trace.batches if b.engine_id in ("vdb-search0", "rerank0")]
    assert gpu and all(b.device_ms is not None and b.device_ms > 0 for b in gpu)
    assert {b.instance_id for b in gpu} == {0, 1}
    assert _check_outputs(rt, backend) > 0


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
