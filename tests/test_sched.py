"""The native engine queue (csrc/tsv_sched.cpp, `sched.TopoQueue`) against the Python mirror of
the reference's form_batch_topo (runtime.py:208-261) over random queues: every batch formed,
dispatched and committed in turn, through to an empty queue. Host-only (no GPU)."""
from __future__ import annotations

import random

import pytest

from paper_2407_00326_b200 import runtime as R
from paper_2407_00326_b200.graph import EGraph, MetadataProfile, PrimitiveKind, PrimitiveNode
from paper_2407_00326_b200.sched import TopoQueue

KINDS = [PrimitiveKind.SEARCHING, PrimitiveKind.RERANKING, PrimitiveKind.EMBEDDING,
         PrimitiveKind.PARTIAL_PREFILLING, PrimitiveKind.DECODING]


def random_tasks(rng: random.Random, n_queries: int, max_nodes: int):
    tasks = []
    seq = 0
    for qi in range(n_queries):
        qid = f"q{rng.randrange(1000):03d}-{qi}"
        g = EGraph(query_id=qid)
        ctx = R.QueryContext(query_id=qid, graph=g, arrival_ms=0.0)
        for j in range(rng.randint(1, max_nodes)):
            nid = f"n{rng.randrange(50):02d}_{j}"
            kind = rng.choice(KINDS)
            node = PrimitiveNode(nid, kind, MetadataProfile())
            g.nodes[nid] = node
            g.depth[nid] = rng.randrange(4)
            # integer-valued and fractional loads; ties in arrival across queries
            loads = [float(rng.choice([1, 1, 2, 0.5, 3.25, 7])) for _ in range(rng.randint(0, 12))]
            t = R.NodeTask(ctx=ctx, node=node, arrival_ms=float(rng.choice([0, 1, 1, 2.5, 3])),
                           seq=seq, loads=loads)
            t.next_request = rng.randint(0, len(loads)) if rng.random() < 0.2 else 0
            seq += 1
            tasks.append(t)
    return tasks


def enc(plan, idx):
    return ([(idx[id(t)], n) for t, n in plan.entries], plan.load, plan.phase if plan else None)


@pytest.mark.parametrize("seed", range(40))
def test_native_queue_matches_mirror_to_drain(seed):
    # two independent copies of the same queue state: one for the mirror, one for the queue
    rng = random.Random(seed)
    py = random_tasks(rng, rng.randint(1, 8), 6)
    rng2 = random.Random(seed)
    mirror = random_tasks(rng2, rng2.randint(1, 8), 6)
    idx_py = {id(t): i for i, t in enumerate(py)}
    idx_m = {id(t): i for i, t in enumerate(mirror)}
    q = TopoQueue(R.EPS)
    for t in mirror:
        q.push(t)
    queue = list(py)
    for step in range(500):
        cap = rng.choice([1.0, 2.0, 4.0, 7.5, 16.0, 64.0])
        a = R.form_batch_topo(queue, cap, 0.0)
        b = q.form(cap)
        assert enc(a, idx_py) == enc(b, idx_m), (seed, step)
        if not a:
            break
        for (ta, n), (tb, m) in zip(a.entries, b.entries):
            ta.next_request += n
            tb.next_request += m
        queue = [t for t in queue if t.pending() > 0]
        q.commit(b.entries)
    else:
        pytest.fail("queue did not drain")
    assert all(t.pending() <= 0 for t in py)
    q.close()


def test_native_queue_grows_entry_buffers():
    rng = random.Random(7)
    g = EGraph(query_id="q")
    ctx = R.QueryContext(query_id="q", graph=g, arrival_ms=0.0)
    q = TopoQueue(R.EPS)
    tasks = []
    for j in range(300):  # 300 one-request tasks at one depth: one batch of 300 entries
        node = PrimitiveNode(f"n{j:04d}", PrimitiveKind.SEARCHING, MetadataProfile())
        g.nodes[node.node_id] = node
        g.depth[node.node_id] = 0
        t = R.NodeTask(ctx=ctx, node=node, arrival_ms=rng.random(), seq=j, loads=[1.0])
        tasks.append(t)
        q.push(t)
    plan = q.form(1000.0)
    assert [t.node.node_id for t, _ in plan.entries] == sorted(t.node.node_id for t in tasks)
    assert plan.load == 300.0
    for t, n in plan.entries:
        t.next_request += n
    q.commit(plan.entries)
    assert len(q) == 0 and not q.form(1000.0)
    q.close()
