"""The INTEGRATION.md binding works against the reference's own Simulator.

Runs only where the reference is importable (the development container); a recording stub
stands in for the GPU backend (it returns the profile latency, as timing="profile" does).
The bound simulator must reproduce the plain reference trace exactly, and every
vdb-search0 / rerank0 batch must have gone through the backend."""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not available")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF))
    import teola_sim.engines as E
    import teola_sim.optimizer as O
    import teola_sim.runtime as rt
    from teola_sim.workflow import QueryConfig
    from teola_sim.workloads import AppKind, build_app_template

    return E, O, rt, QueryConfig, AppKind, build_app_template


class RecordingBackend:
    """Stand-in with RetrievalBackend's interface; records what it was asked to run."""

    def __init__(self, latency):
        self.latency = latency
        self.batches = []
        self.completed = []

    def serves(self, profile):
        return profile.engine_id in ("vdb-search0", "rerank0")

    def execute(self, profile, plan, t, instance):
        self.batches.append((profile.engine_id, instance.instance_id,
                             [(task.node_id, n) for task, n in plan.entries]))
        return self.latency(profile, plan.load), None

    def on_complete(self, ctx, node):
        self.completed.append(node.node_id)


def _bound_simulator(rt, select_instance):
    # verbatim shape of INTEGRATION.md §2
    class B200Simulator(rt.Simulator):
        def __init__(self, engines, options=None, backend=None):
            super().__init__(engines, options)
            self.backend = backend

        def _dispatch(self, state, plan, t):
            self._instance = select_instance(state.instances, state.profile.category, t)
            return super()._dispatch(state, plan, t)

        def _execute(self, profile, plan, t):
            if not plan.entries:
                raise rt.CapacityExceeded("empty batch")
            if self.backend is not None and plan.phase == rt.PHASE_GENERAL \
                    and self.backend.serves(profile):
                duration, _ = self.backend.execute(profile, plan, t, self._instance)
                return duration, [(task, n, t + duration) for task, n in plan.entries], 0.0
            return super()._execute(profile, plan, t)

        def on_primitive_complete(self, ctx, node_id, now):
            self.backend.on_complete(ctx, ctx.graph.nodes[node_id])
            return super().on_primitive_complete(ctx, node_id, now)

    return B200Simulator


@pytest.mark.parametrize("app", ["ADVANCED_RAG_QA", "CONTEXTUAL_RETRIEVAL", "NAIVE_RAG_QA"])
def test_binding_preserves_reference_trace(ref, app):
    E, O, rt, QueryConfig, AppKind, build = ref
    es = E.load_profiles("default")
    kind = getattr(AppKind, app)
    graphs = [O.compile_query(build(kind), QueryConfig(query_id=f"q{i}"), es) for i in range(3)]
    plain = rt.Simulator(es)
    for i, g in enumerate(graphs):
        plain.submit_query(g, 25.0 * i)
    want = plain.run().rows()

    backend = RecordingBackend(E.latency)
    sim = _bound_simulator(rt, E.select_instance)(es, backend=backend)
    for i, g in enumerate(graphs):
        sim.submit_query(g.clone(), 25.0 * i)
    assert sim.run().rows() == want
    ran = {n for _, _, entries in backend.batches for n, _ in entries}
    expect = {b_node for b in plain.trace.batches if b.engine_id in ("vdb-search0", "rerank0")
              for b_node in b.node_ids}
    assert ran == expect and ran
