"""Real-time stream/event execution of e-graphs, and CUDA-graph capture of a search.

Replaces the reference's threaded execution mode (pkg/src/teola_sim/threaded.py:130-182:
one Python thread per engine forming batches under a lock and sleeping `latency / speed`).
Here one host thread runs the same two-tier scheduler as the simulator (the mirror in
runtime.py: per-query graph tier, form_batch_topo / form_batch_blind, select_instance), but:

  * GPU engines (`vdb-search0`, `rerank0`) launch their batch on the chosen replica's CUDA
    stream and return immediately; the batch completes when its end event completes
    (polled, no host blocking), so batches on different replicas run concurrently and stage
    pipelines of different queries overlap;
  * Aggregate joins are stream-ordered (cudaStreamWaitEvent + concat/K4 in the backend), so
    no host synchronisation sits between search stages and the rerank that consumes them;
  * modelled engines (LLM, embedding, ingest, web) complete after their profile latency in
    wall time divided by `speed` (the threaded mode's semantics).

Timestamps in the trace are wall-clock milliseconds x speed since start (threaded.py:58-59).

`CapturedSearch` captures a fixed-shape search (query staging + fused scan + merge) into a
CUDA graph and replays it: one graph launch per batch instead of three kernel launches, for
the launch-bound small-batch retrieval of per-query workflows.
"""

from __future__ import annotations

import heapq
import math
import time

import torch

from .engines import EngineSet
from ._native import PrivateStream
from .errors import ConfigParse
from .graph import CONTROL_KINDS
from .runtime import BatchRecord, RuntimeOptions, Simulator


class StreamRuntime(Simulator):
    """Wall-clock execution of submitted e-graphs; retrieval batches complete on CUDA events.

    Edges cost nothing: like the reference's threaded mode (threaded.py:108-128: a completed
    node dispatches its ready children at once), there is no modelled Ray hop here — a
    transfer that really happens (a query's index pulled to another replica) is a peer copy on
    the device, inside the measured batch.

    stream_order=True (default) maps the reference's pre-scheduling (runtime.py:419-454) onto
    CUDA stream order: a GPU batch completes *logically* when it is launched, so the consumers
    that run on the device (the next Searching stage, the Aggregate join, Reranking) are
    dispatched right away and their kernels queue behind the producer's on the replica stream
    (cross-replica consumers wait on the producer's event; backend.py). Consumers on modelled
    engines (LLM, embedding, ...) are only released once every device batch upstream of them
    has finished (its end event), so nothing modelled starts before its GPU input exists. The
    trace's `complete` event of a GPU node is its launch; BatchRecord keeps the device-measured
    time of every batch and `device_done` events mark the real completions."""

    def __init__(self, engines: EngineSet, backend, options: RuntimeOptions | None = None,
                 speed: float = 1.0, poll_us: float = 20.0, timeout_s: float = 60.0,
                 stream_order: bool = True, busy_poll: bool = True, affinity: bool = True,
                 fuse_chains: bool = True, queue_on_stream: bool = False):
        """busy_poll: while device batches are in flight, poll their events without sleeping
        (an OS sleep of 20 us lasts ~60-80 us, which would add to every device -> host hop);
        the loop sleeps only when nothing is in flight and the next event is in the future."""
        super().__init__(engines, options, backend=backend)
        self.speed = speed
        self.busy_poll = busy_poll
        self.affinity = affinity
        self.fuse_chains = fuse_chains and stream_order
        # queue_on_stream: a GPU replica takes its next batch as soon as the previous one is
        # launched (the replica's stream still runs them one at a time). Off by default: with
        # 30 concurrent C3 queries it made batches smaller and the retrieval tail longer (4.0 vs
        # 3.0 ms, scripts/stream_probe.py) — each batch costs ~0.14 ms of host time, so batching
        # behind the previous launch's completion pays
        self.queue_on_stream = queue_on_stream and stream_order
        self._chained: dict[tuple[str, str], object] = {}  # (query, rerank node) -> end event
        self._chain_nodes: dict[int, list] = {}  # id(end event) -> fused rerank nodes
        self.poll_s = poll_us * 1e-6
        self.timeout_s = timeout_s
        self.stream_order = stream_order
        self._t0 = None
        self._inflight: list[tuple] = []  # (end_event, start_event, state, instance, plan, t)
        self._node_events: dict[tuple[str, str], list] = {}  # (query, node) -> end events
        self._parked: list[tuple] = []  # (ctx, node_id, events) waiting for device inputs
        self.device_done: list[tuple[float, str, str]] = []  # (ms, query, node)

    def _wall(self) -> float:
        return (time.perf_counter() - self._t0) * 1000.0 * self.speed

    def _edge_delay(self, graph, e) -> float:
        return 0.0

    def _gpu(self, node) -> bool:
        return (self.backend is not None and node.meta.engine_id in self.engines
                and self.backend.serves(self.engines[node.meta.engine_id].profile))

    def _upstream_events(self, ctx, nid: str, seen=None) -> list:
        """Device end events a node's inputs still depend on: its GPU producers' batches, and
        through control nodes (Aggregate) their producers'."""
        seen = set() if seen is None else seen
        out = []
        for e in ctx.graph.edges:
            if e.dst != nid or e.src in seen:
                continue
            seen.add(e.src)
            src = ctx.graph.nodes[e.src]
            out += self._node_events.get((ctx.query_id, e.src), [])
            if src.kind in CONTROL_KINDS:
                out += self._upstream_events(ctx, e.src, seen)
        return out

    def _node_ready(self, ctx, nid: str, t: float) -> None:
        end = self._chained.pop((ctx.query_id, nid), None)
        if end is not None:
            # a Reranking node whose result the fused chain launch already computes: it
            # completes in stream order, without a batch of its own (its consumers on modelled
            # engines wait for the launch's end event)
            node = ctx.graph.nodes[nid]
            self._node_events.setdefault((ctx.query_id, nid), []).append(end)
            if ctx.stats[nid].ready_ms is None:
                ctx.stats[nid].ready_ms = t
            self._emit(t, ctx, node, "enqueue")
            ctx.stats[nid].first_start_ms = t
            self._emit(t, ctx, node, "start")
            self.on_primitive_complete(ctx, nid, t)
            return
        node = ctx.graph.nodes[nid]
        if self.stream_order and node.kind not in CONTROL_KINDS and not self._gpu(node):
            pending = [ev for ev in self._upstream_events(ctx, nid) if not ev.query()]
            if pending:
                self._parked.append((ctx, nid, pending))
                return
        super()._node_ready(ctx, nid, t)

    # GPU batches: launch and return; completion is discovered by polling the end event.
    def _dispatch(self, state, plan, t):
        profile = state.profile
        if not (self.backend is not None and self.backend.serves(profile)
                and plan.phase == "general"):
            return super()._dispatch(state, plan, t)
        from .engines import select_instance

        instance = self._affine_instance(state, plan, t) if self.affinity else None
        if instance is None:
            instance = select_instance(state.instances, profile.category, t)
        assert instance is not None
        chain = self._chain_reranks(plan) if (self.fuse_chains and profile.category == "search") else None
        launched = None
        if chain is not None and hasattr(self.backend, "launch_chain"):
            launched = self.backend.launch_chain(profile, plan, instance, chain)
        if launched is not None:
            start, end = launched
            for (task, _), rr in zip(plan.entries, chain):
                self._chained[(task.ctx.query_id, rr.node_id)] = end
            self._chain_nodes[id(end)] = [(task.ctx.query_id, rr.node_id)
                                          for (task, _), rr in zip(plan.entries, chain)]
        else:
            start, end = self.backend.launch(profile, plan, instance)
        # busy until the end event fires (or, queued on the stream, free for the next batch)
        instance.busy_until = t if self.queue_on_stream else math.inf
        instance.executed_requests += sum(n for _, n in plan.entries)
        for task, n in plan.entries:
            task.next_request += n
            self._emit(t, task.ctx, task.node, "batch")
            if task.ctx.stats[task.node_id].first_start_ms is None:
                task.ctx.stats[task.node_id].first_start_ms = t
                self._emit(t, task.ctx, task.node, "start")
            self._node_events.setdefault((task.ctx.query_id, task.node_id), []).append(end)
            if self.stream_order:  # consumers queue behind this batch in stream order
                self._push(t, self._REQ_DONE, (task, n))
        self._drop_drained(state, plan)
        self._inflight.append((end, start, state, instance, plan, t))

    def _chain_reranks(self, plan):
        """Fused dispatch of a search -> rerank chain (the contextual workflow's stage pair):
        for every entry, the whole Searching node (one query vector, a per-query index) whose
        only consumer is a Reranking node on a backend engine, fed by nothing else — the
        rerank's result can be computed by the same launch (tsv_search_rerank_segmented).
        Returns the rerank nodes in entry order, or None when any entry does not qualify."""
        out = []
        for task, n in plan.entries:
            node, g = task.node, task.ctx.graph
            if task.next_request != 0 or n != len(task.loads) or node.meta.batch_items != 1:
                return None
            if not any(e.dst == node.node_id and e.key == "index" for e in g.edges):
                return None
            consumers = [e.dst for e in g.edges if e.src == node.node_id]
            if len(consumers) != 1:
                return None
            rr = g.nodes[consumers[0]]
            if rr.kind.value != "Reranking" or not self._gpu(rr):
                return None
            feeds = [e for e in g.edges if e.dst == rr.node_id and e.key is not None]
            if any(e.src != node.node_id for e in feeds):
                return None
            out.append(rr)
        return out

    def _affine_instance(self, state, plan, t):
        """Index-location affinity (the reference picks the least-loaded replica,
        engines.py:156-164, blind to data placement): an idle replica on the GPU that holds the
        per-query indexes of most of the batch's entries, so no segment is pulled over NVLink.
        Ties and batches without per-query indexes keep select_instance's choice."""
        home = getattr(self.backend, "home", None)
        if home is None or len(state.instances) < 2:
            return None
        idle = [i for i in state.instances if i.idle(t)]
        if len(idle) < 2:
            return None
        votes: dict[int, int] = {}
        for task, n in plan.entries:
            if any(e.dst == task.node_id and e.key == "index" for e in task.ctx.graph.edges) or \
                    task.node.kind.value == "Reranking":
                r = home(task.ctx.query_id)
                votes[r] = votes.get(r, 0) + n
        if not votes:
            return None
        n_rep = len(self.backend.replicas)
        best = max(votes.items(), key=lambda kv: (kv[1], -kv[0]))[0]
        on_home = [i for i in idle if i.instance_id % n_rep == best]
        if not on_home:
            return None
        return min(on_home, key=lambda i: (i.executed_requests, i.instance_id))

    def _poll(self, t: float) -> bool:
        progressed = False
        if self._parked:
            still = []
            for ctx, nid, evs in self._parked:
                evs = [ev for ev in evs if not ev.query()]
                if evs:
                    still.append((ctx, nid, evs))
                else:
                    Simulator._node_ready(self, ctx, nid, t)
                    progressed = True
            self._parked = still
        done, still = [], []
        for x in self._inflight:
            (done if x[0].query() else still).append(x)
        if not done:
            return progressed
        self._inflight = still
        for end, start, state, instance, plan, t0 in done:
            if not self.queue_on_stream:
                instance.busy_until = t
            device_ms = start.elapsed_time(end)
            for task, n in plan.entries:
                if not self.stream_order:
                    self._push(t, self._REQ_DONE, (task, n))
                self.device_done.append((t, task.ctx.query_id, task.node_id))
            for qid, rr_id in self._chain_nodes.pop(id(end), []):
                self.device_done.append((t, qid, rr_id))
            self._push(t, self._BATCH_DONE, (state.profile.engine_id, instance.instance_id, 0.0))
            self.trace.batches.append(BatchRecord(state.profile.engine_id, instance.instance_id,
                                                  t0, t, plan.load, self._cap(state), plan.phase,
                                                  plan.node_ids(), device_ms))
        return True

    def run(self, until: float | None = None):
        self._t0 = time.perf_counter()
        deadline = time.perf_counter() + self.timeout_s
        while self._events or self._inflight or self._parked:
            if time.perf_counter() > deadline:
                raise TimeoutError("stream runtime did not quiesce")
            t = self._wall()
            progressed = self._poll(t)
            while self._events and self._events[0][0] <= t:
                ts, _, tag, payload = heapq.heappop(self._events)
                self.now = ts
                self._handle(tag, payload, ts)
                progressed = True
            for eid in sorted(self._dirty):
                self._try_form(eid, t)
            self._dirty.clear()
            if not progressed and not (self.busy_poll and (self._inflight or self._parked)):
                nxt = self._events[0][0] if self._events else math.inf
                wait_s = min(self.poll_s, max(0.0, (nxt - t) / 1000.0 / self.speed))
                if wait_s > 0:
                    time.sleep(wait_s)
        if self.backend is not None:
            self.backend.finish()
        return self.trace


def run_streamed(engines: EngineSet, graphs_with_arrivals, backend,
                 options: RuntimeOptions | None = None, speed: float = 1.0):
    """Submit (graph, arrival_ms) pairs and execute them in real time on CUDA streams."""
    rt = StreamRuntime(engines, backend, options, speed=speed)
    for g, arrival in graphs_with_arrivals:
        rt.submit_query(g, arrival, arrival_ms=arrival)
    return rt, rt.run()


def _same_shape(t: torch.Tensor, captured: torch.Tensor, name: str) -> None:
    """Replays take exactly the captured shapes (copy_ would broadcast a mismatch silently)."""
    if tuple(t.shape) != tuple(captured.shape):
        raise ConfigParse(f"{name}: shape {tuple(t.shape)} differs from the captured "
                          f"{tuple(captured.shape)}")


class CapturedSearch:
    """A fixed-shape search captured in a CUDA graph.

    search(q) copies q into the captured input buffer and replays the graph; results land in
    the captured output buffers (returned, valid until the next call)."""

    def __init__(self, index, batch: int, k: int, row_range: tuple[int, int] | None = None,
                 id_offset: int = 0, dtype=torch.bfloat16, warmup: int = 2):
        self.index = index
        dev = index.device
        self.q = torch.zeros((batch, index.dim), dtype=dtype, device=dev)
        self.scores = torch.empty((batch, k), dtype=torch.float32, device=dev)
        self.ids = torch.empty((batch, k), dtype=torch.int32, device=dev)
        self.k = k
        self.row_range = row_range
        self.id_offset = id_offset
        # a library-created stream kept for the graph's lifetime (never shared through torch's
        # stream pool): its per-stream scratch in the index is this graph's alone
        self._stream = PrivateStream(dev.index)
        stream = self._stream.stream
        with torch.cuda.stream(stream):
            for _ in range(warmup):  # grows the per-stream workspace before capture
                self._run(stream)
        stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=stream, capture_error_mode="thread_local"):
            self._run(torch.cuda.current_stream(dev))

    def _run(self, stream):
        self.index.search(self.q, self.k, row_range=self.row_range, id_offset=self.id_offset,
                          stream=stream, out=(self.scores, self.ids))

    def search(self, q: torch.Tensor):
        _same_shape(q, self.q, "queries")
        self.q.copy_(q)
        self.graph.replay()
        return self.scores, self.ids


class CapturedRetrieval:
    """The advanced-RAG retrieval chain captured in one CUDA graph: Searching
    over `questions * expansions` expanded queries (top-k_search each), the Aggregate join of a
    question's expansions (a view: candidates in slice order, optimizer.py:620-661) and
    Reranking of those candidates against the question (dedup, top-k_rerank;
    optimizer.py:199-218). One graph replay replaces the chain's 6-8 kernel launches (k > 32
    search: sample pass, merges, candidate pass, select, gated fallback; K3) and their host
    issue cost.

    run(qx, qq) copies the expanded queries [questions * expansions, dim] and the questions
    [questions, dim] into the captured buffers and replays; returns the reranked (scores, ids)
    buffers (valid until the next call). The graph owns a private stream, so its per-stream
    workspace in the index is not shared with other callers."""

    def __init__(self, index, questions: int, expansions: int, k_search: int, k_rerank: int,
                 dtype=torch.bfloat16, warmup: int = 2):
        self.index = index
        dev = index.device
        self.questions, self.expansions = questions, expansions
        self.k_search, self.k_rerank = k_search, k_rerank
        self.qx = torch.zeros((questions * expansions, index.dim), dtype=dtype, device=dev)
        self.qq = torch.zeros((questions, index.dim), dtype=dtype, device=dev)
        self.s_s = torch.empty((questions * expansions, k_search), dtype=torch.float32, device=dev)
        self.s_i = torch.empty((questions * expansions, k_search), dtype=torch.int32, device=dev)
        self.r_s = torch.empty((questions, k_rerank), dtype=torch.float32, device=dev)
        self.r_i = torch.empty((questions, k_rerank), dtype=torch.int32, device=dev)
        # a library-created stream kept for the graph's lifetime (never shared through torch's
        # stream pool): its per-stream scratch in the index is this graph's alone
        self._stream = PrivateStream(dev.index)
        stream = self._stream.stream
        with torch.cuda.stream(stream):
            for _ in range(warmup):  # grows the per-stream workspace before capture
                self._run(stream)
        stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=stream, capture_error_mode="thread_local"):
            self._run(torch.cuda.current_stream(dev))

    def _run(self, stream):
        self.index.search(self.qx, self.k_search, stream=stream, out=(self.s_s, self.s_i))
        cand = self.s_i.view(self.questions, self.expansions * self.k_search)  # Aggregate
        self.index.rerank(self.qq, cand, self.k_rerank, stream=stream, out=(self.r_s, self.r_i))

    def run(self, qx: torch.Tensor, qq: torch.Tensor):
        _same_shape(qx, self.qx, "expanded queries")
        _same_shape(qq, self.qq, "questions")
        self.qx.copy_(qx)
        self.qq.copy_(qq)
        self.graph.replay()
        return self.r_s, self.r_i


class CapturedContextual:
    """The contextual-retrieval chain captured in one CUDA graph: each query
    searches its own per-query index segment (segmented Searching, top-k_search; the
    per-query indexes of workloads.py:95-97 built by each query's Ingestion) and its hits are
    reranked against it (Reranking, dedup, top-k_rerank). Segment layout is fixed at capture.

    fused=None (default) runs the chain as ONE kernel (tsv_search_rerank_segmented: the
    segment's rows are gathered once and scored against the query and the rerank question in
    the same pass) whenever every segment has <= 1024 rows on a bf16 arena; fused=False keeps the primitive-by-primitive chain (normalise + scan + merge
    + rerank: its item list lives in a pinned buffer owned by the index).

    run(q) copies the queries into the captured buffer and replays; returns the reranked
    (scores, ids) buffers, ids being arena rows (valid until the next call)."""

    def __init__(self, index, q_offsets, row_ranges, k_search: int, k_rerank: int,
                 dtype=torch.bfloat16, warmup: int = 2, fused: bool | None = None):
        self.index = index
        dev = index.device
        b = int(q_offsets[-1])
        self.q_offsets, self.row_ranges = list(q_offsets), list(row_ranges)
        self.k_search, self.k_rerank = k_search, k_rerank
        max_rows = max((e - a for a, e in self.row_ranges), default=0)
        can_fuse = (index.storage in ("bf16", "bf16_tiled") and index.dim <= 2048
                    and 0 < max_rows <= 1024 and k_rerank <= k_search)
        if fused and not can_fuse:
            raise ConfigParse("fused contextual chain needs a bf16 arena (dim <= 2048) and "
                              "segments of 1..1024 rows")
        self.fused = can_fuse if fused is None else bool(fused)
        self.max_rows = max_rows
        self.q = torch.zeros((b, index.dim), dtype=dtype, device=dev)
        self.s_s = torch.empty((b, k_search), dtype=torch.float32, device=dev)
        self.s_i = torch.empty((b, k_search), dtype=torch.int32, device=dev)
        self.r_s = torch.empty((b, k_rerank), dtype=torch.float32, device=dev)
        self.r_i = torch.empty((b, k_rerank), dtype=torch.int32, device=dev)
        rows = []
        for sidx, (a, e) in enumerate(self.row_ranges):
            rows += [(a, e)] * (self.q_offsets[sidx + 1] - self.q_offsets[sidx])
        self.q_rows = torch.tensor(rows, dtype=torch.int64).reshape(b, 2).to(dev)
        # a library-created stream kept for the graph's lifetime (never shared through torch's
        # stream pool): its per-stream scratch in the index is this graph's alone
        self._stream = PrivateStream(dev.index)
        stream = self._stream.stream
        with torch.cuda.stream(stream):
            for _ in range(warmup):  # grows the per-stream workspace before capture
                self._run(stream)
        stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=stream, capture_error_mode="thread_local"):
            self._run(torch.cuda.current_stream(dev))

    def _run(self, stream):
        if self.fused:
            self.index.search_rerank_segmented(self.q, self.q_rows, self.max_rows, self.k_search,
                                               self.k_rerank, local_ids=False, stream=stream,
                                               out_search=(self.s_s, self.s_i),
                                               out_rerank=(self.r_s, self.r_i))
            return
        self.index.search_segmented(self.q, self.q_offsets, self.row_ranges, self.k_search,
                                    local_ids=False, stream=stream, out=(self.s_s, self.s_i))
        self.index.rerank(self.q, self.s_i, self.k_rerank, stream=stream,
                          out=(self.r_s, self.r_i))

    def run(self, q: torch.Tensor):
        _same_shape(q, self.q, "queries")
        self.q.copy_(q)
        self.graph.replay()
        return self.r_s, self.r_i
