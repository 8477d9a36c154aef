"""RetrievalBackend: executes Searching / Reranking batch plans on B200 GPUs.

This is what `Simulator._execute` hands a plan to for the engines it is bound to (in the
reference the same call returns `latency(profile, load)`; pkg/src/teola_sim/runtime.py:653-655).
Engine replicas map to GPUs (`EngineProfile.instances`, chosen by `select_instance`,
engines.py:156-164). Data flows through the object store exactly along the graph's edges:

  Embedding (modeled)   -> query vectors [items, D] for the node's slice (seeded synthetic)
  Ingestion (modeled)   -> chunk vectors appended to the replica's device arena; the query's
                           index is a contiguous arena segment (all ingest stages of a query
                           write into one reserved segment at their slice offsets)
  Searching (GPU, K1/K2)-> per query top-k (scores, chunk ids), query-major, for the stage's
                           slice; a whole topology-aware batch is ONE segmented launch, each
                           entry searching its own query's index segment (or the resident
                           global corpus when the node has no index input)
  Aggregate (K4 / cat)  -> stage results concatenated in slice order (optimizer.py:620-661)
  Reranking (GPU, K3)   -> candidate chunks scored against the question vector, deduplicated,
                           top_k kept; requests (candidates) split across batches are merged
                           with K4 when the node completes

Timing: "profile" keeps the profile latency as the batch duration (reference-identical
traces); "measured" returns the device time of the batch's launches (CUDA events on the
replica's stream). Either way the kernels run and the results are real.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import torch

from . import _native
from .engines import EngineProfile, latency
from .errors import CapacityExceeded, ConfigParse
from .graph import PrimitiveKind, PrimitiveNode
from .index import DeviceIndex, merge_topk, normalize_rows

TIMING_PROFILE = "profile"
TIMING_MEASURED = "measured"


def _seed(*parts) -> int:
    h = hashlib.sha256("|".join(str(p) for p in parts).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


class SyntheticData:
    """Deterministic stand-ins for the outputs of the modeled (non-GPU) primitives.

    Rows are generated in blocks of 64 seeded from (query id, key, block), so any stage split
    reproduces exactly the rows the unsplit node would, at the cost of the rows it needs. A
    `planted` fraction of query vectors are near-copies of one of the query's own chunks (the
    retrieval target), mirroring the bench's planted-neighbour queries."""

    BLOCK = 64

    def __init__(self, dim: int, seed: int = 0, planted: float = 0.5, noise: float = 0.05):
        self.dim = dim
        self.seed = seed
        self.planted = planted
        self.noise = noise

    def _rows(self, device, tag: tuple, lo: int, hi: int) -> torch.Tensor:
        if hi <= lo:
            return torch.empty((0, self.dim), device=device)
        parts = []
        for b in range(lo // self.BLOCK, (hi - 1) // self.BLOCK + 1):
            g = torch.Generator(device=device).manual_seed(_seed(self.seed, *tag, b))
            blk = torch.randn((self.BLOCK, self.dim), generator=g, device=device)
            a = max(lo, b * self.BLOCK) - b * self.BLOCK
            e = min(hi, (b + 1) * self.BLOCK) - b * self.BLOCK
            parts.append(blk[a:e])
        return torch.cat(parts) if len(parts) > 1 else parts[0]

    def chunks(self, device, query_id: str, key: str, lo: int, hi: int, total: int) -> torch.Tensor:
        return normalize_rows(self._rows(device, ("chunks", query_id, key), lo, hi).contiguous())

    def queries(self, device, query_id: str, key: str, lo: int, hi: int, total: int,
                n_chunks: int | None = None, chunk_key: str | None = None) -> torch.Tensor:
        q = self._rows(device, ("queries", query_id, key), lo, hi).clone()
        if n_chunks and chunk_key is not None and self.planted > 0:
            m = int(round(total * self.planted))
            g = torch.Generator(device="cpu").manual_seed(_seed(self.seed, "plant", query_id))
            rows = torch.randint(0, n_chunks, (m,), generator=g).tolist()
            for i in range(lo, min(hi, m)):
                base = self._rows(device, ("chunks", query_id, chunk_key), rows[i], rows[i] + 1)
                q[i - lo] = base[0] + self.noise * q[i - lo]
        return normalize_rows(q.contiguous())

    def question(self, device, query_id: str) -> torch.Tensor:
        return normalize_rows(self._rows(device, ("question", query_id), 0, 1).contiguous())


@dataclass
class IndexSegment:
    """A query's per-query index: rows [row_beg, row_end) of one replica's arena."""

    replica: int
    row_beg: int
    row_end: int
    filled: int = 0


@dataclass
class SearchResult:
    """Searching output for queries [q_lo, q_hi) of the node: (scores, ids) [n, k] on device;
    ids are chunk ids within the query's index (or global corpus ids). `ready` is recorded on
    the producing replica stream; consumers on other streams wait on it."""

    scores: torch.Tensor
    ids: torch.Tensor
    q_lo: int
    q_hi: int
    slice_of: tuple[int, int, int] | None = None
    ready: torch.cuda.Event | None = None
    replica: int = 0


@dataclass
class LaunchRecord:
    """Per-batch device record (SURVEY.md §5 tracing): what one retrieval batch moved and
    computed, and how long the device took."""

    engine_id: str
    replica: int
    kind: str          # "search" | "rerank"
    queries: int       # queries (search) or questions (rerank)
    rows: int          # corpus rows scanned (search) or candidate rows gathered (rerank)
    k: int
    dim: int
    bytes: int         # algorithmic bytes: rows + queries read, results written
    flops: int         # algorithmic flops (2 per multiply-add)
    start: object = None
    end: object = None

    @property
    def device_ms(self) -> float:
        return self.start.elapsed_time(self.end)


@dataclass
class Replica:
    device: torch.device
    stream: torch.cuda.Stream
    arena: DeviceIndex
    # released index segments: (row_beg, rows, event the reuse must wait for)
    free: list = field(default_factory=list)


class RetrievalBackend:
    """Executes batches of the bound retrieval engines on GPU replicas.

    engines: engine ids to serve (default: every engine of category search/rerank that the
    workflow uses for vector search — `vdb-search0`, `rerank0`). `web0` / `tool0` searches
    stay latency-modeled."""

    def __init__(self, dim: int, devices: list[int] | None = None, arena_rows: int = 1 << 20,
                 engines=("vdb-search0", "rerank0"), timing: str = TIMING_PROFILE,
                 data: SyntheticData | None = None, metric: str = "cosine",
                 global_index=None, release_segments: bool = True):
        """global_index: the resident corpus searched by Searching nodes that have no per-query
        index input — a DeviceIndex, or a ShardedIndex spanning several devices (shards
        searched concurrently, merged on its root device).
        release_segments: a finished query's index segments return to the arena's free list
        and its device results are dropped (False keeps them for inspection, e.g. tests)."""
        self.release_segments = release_segments
        if timing not in (TIMING_PROFILE, TIMING_MEASURED):
            raise ConfigParse(f"unknown timing mode {timing!r}")
        _native.load()
        self.dim = dim
        self.timing = timing
        self.engines = set(engines)
        self.data = data or SyntheticData(dim)
        self.global_index = global_index
        devs = devices if devices is not None else [torch.cuda.current_device()]
        self.replicas = []
        for d in devs:
            dev = torch.device("cuda", d)
            with torch.cuda.device(dev):
                self.replicas.append(Replica(dev, torch.cuda.Stream(dev),
                                             DeviceIndex(dim, arena_rows, metric=metric, device=d)))
        self.segments: dict[tuple[str, str, int], IndexSegment] = {}  # (query, key, replica)
        # (query id, node id) -> [(first request, scores, ids)] of batches run so far
        self.acc: dict[tuple[str, str], list] = {}
        self._edge_index: dict[int, tuple] = {}  # id(graph) -> (graph, edge count, in-edges)
        self._waited: dict = {}  # (replica, event) pairs already waited in the current launch
        self.launches = 0
        self.device_ms_total = 0.0
        self.records: list[LaunchRecord] = []

    # -- binding ---------------------------------------------------------------------
    def serves(self, profile: EngineProfile) -> bool:
        return profile.engine_id in self.engines and profile.category in ("search", "rerank")

    def replica_for(self, instance) -> Replica:
        iid = 0 if instance is None else instance.instance_id
        return self.replicas[iid % len(self.replicas)]

    def home(self, query_id: str) -> int:
        return _seed("home", query_id) % len(self.replicas)

    # -- graph-tier hooks --------------------------------------------------------------
    def on_submit(self, ctx) -> None:
        """The question vector a query's Reranking scores against stands for the output of a
        modelled embedding: materialise it once, on the query's home replica, outside every
        retrieval batch."""
        rep = self.replicas[self.home(ctx.query_id)]
        if any(n.kind is PrimitiveKind.RERANKING and n.meta.engine_id in self.engines
               for n in ctx.graph.nodes.values()):
            with self._on(rep):
                qv = self.data.question(rep.device, ctx.query_id)
                ctx.data[("__question__", None)] = (qv, self._record(rep))

    def on_query_done(self, ctx) -> None:
        """A query finished: its per-query index segments go back to their replicas' free
        lists (reused once every stream that may still read them has passed this point), and
        its device results are dropped."""
        if not self.release_segments:
            return
        mine = [key for key in self.segments if key[0] == ctx.query_id]
        for key in mine:
            seg = self.segments.pop(key)
            rep = self.replicas[seg.replica]
            evs = []
            for r in self.replicas:
                ev = torch.cuda.Event()
                ev.record(r.stream)
                evs.append(ev)
            rep.free.append((seg.row_beg, seg.row_end - seg.row_beg, evs))
        for key in [k for k in self.acc if k[0] == ctx.query_id]:
            del self.acc[key]
        self._edge_index.pop(id(ctx.graph), None)
        ctx.data.clear()

    def on_complete(self, ctx, node: PrimitiveNode) -> None:
        """Materialise the device data a completed node produces."""
        kind = node.kind
        if kind is PrimitiveKind.INGESTION:
            for key, p in node.meta.outputs.items():
                self._ingest(ctx, node, key, p.items)
        elif kind is PrimitiveKind.EMBEDDING:
            # Query vectors are materialised here, when the (modelled) embedding finishes, so
            # their generation is not part of the Searching batch that consumes them.
            for key, p in node.meta.outputs.items():
                lo, hi, total = node.meta.slice_of.get(key, (0, p.items, p.items))
                n_chunks, chunk_key = self._index_feeding(ctx, node.node_id, key)
                rep = self.replicas[self.home(ctx.query_id)]
                with self._on(rep):
                    vecs = self.data.queries(rep.device, ctx.query_id, key, lo, hi, total,
                                             n_chunks, chunk_key)
                ctx.data[(node.node_id, key)] = ("queries", key, lo, hi, total, vecs,
                                                 self._record(rep))
        elif kind is PrimitiveKind.AGGREGATE:
            key = node.meta.inputs[0]
            parts = [(ctx.data.get((e.src, key)), e.src) for e in ctx.graph.edges
                     if e.dst == node.node_id and e.key == key]
            parts = [p for p, _ in parts if isinstance(p, SearchResult)]
            if parts:
                # Aggregate = concatenation of the stage results in slice order, ordered after
                # every stage's launch (stream waits, no host sync).
                parts.sort(key=lambda r: (r.slice_of or (0,))[0])
                rep = self.replicas[parts[0].replica]
                with self._on(rep):
                    for p_ in parts:
                        if p_.ready is not None:
                            rep.stream.wait_event(p_.ready)
                    res = SearchResult(torch.cat([p_.scores for p_ in parts]),
                                       torch.cat([p_.ids for p_ in parts]),
                                       min(p_.q_lo for p_ in parts), max(p_.q_hi for p_ in parts),
                                       replica=parts[0].replica)
                    res.ready = self._record(rep)
                ctx.data[(node.node_id, key)] = res
        elif kind in (PrimitiveKind.SEARCHING, PrimitiveKind.RERANKING):
            self._finalize(ctx, node)

    def _on(self, rep: Replica):
        """Context: make `rep`'s device and stream current for torch ops and our launches."""
        return _StreamCtx(rep)

    @staticmethod
    def _record(rep: Replica) -> torch.cuda.Event:
        ev = torch.cuda.Event()
        ev.record(rep.stream)
        return ev

    def _index_feeding(self, ctx, emb_id: str, key: str):
        """(chunk count, key) of the per-query index searched with these query vectors."""
        for e in ctx.graph.edges:
            if e.src == emb_id and e.key == key:
                for f in ctx.graph.edges:
                    if f.dst == e.dst and f.key == "index":
                        prod = ctx.graph.nodes[f.src]
                        if f.key in prod.meta.outputs:
                            s_ = prod.meta.slice_of.get(f.key)
                            return (s_[2] if s_ else prod.meta.outputs[f.key].items), f.key
        return None, None

    def warmup(self) -> None:
        """One tiny search / rerank per replica: first-call costs (function attributes,
        workspace growth, driver entry points) stay out of measured batches."""
        for rep in self.replicas:
            with self._on(rep):
                q = torch.zeros((2, self.dim), dtype=torch.bfloat16, device=rep.device)
                q[:, 0] = 1
                first = rep.arena.append(q)
                rep.arena.search_segmented(q, [0, 1, 2], [(first, first + 2)] * 2, 4,
                                           stream=rep.stream)
                rep.arena.search(q, 4, row_range=(first, first + 2), stream=rep.stream)
                cand = torch.tensor([[first, first + 1]] * 2, dtype=torch.int32, device=rep.device)
                rep.arena.rerank(q, cand, 2, stream=rep.stream)
            rep.stream.synchronize()

    def _ingest(self, ctx, node, key, items):
        lo, hi, total = node.meta.slice_of.get(key, (0, items, items))
        r = self.home(ctx.query_id)
        seg = self._segment(ctx.query_id, key, r, total)
        rep = self.replicas[r]
        with self._on(rep):
            rows = self.data.chunks(rep.device, ctx.query_id, key, lo, hi, total)
            dst = rep.arena.data()[seg.row_beg + lo: seg.row_beg + hi]
            dst.copy_(rows.to(torch.bfloat16))
        seg.filled += hi - lo
        ctx.data[(node.node_id, key)] = ("index", key, total)

    def _reserve(self, rep: Replica, total: int) -> int:
        """Arena rows for a new segment: first fit among released segments (after the streams
        that could still read them), else appended at the end of the arena."""
        for j, (beg, n, evs) in enumerate(rep.free):
            if n >= total:
                for ev in evs:
                    rep.stream.wait_event(ev)
                if n == total:
                    rep.free.pop(j)
                else:
                    rep.free[j] = (beg + total, n - total, evs)
                return beg
        first = rep.arena.rows
        if first + total > rep.arena.capacity:
            raise CapacityExceeded(
                f"replica arena full: {first} + {total} rows > {rep.arena.capacity} "
                f"({sum(n for _, n, _ in rep.free)} rows free in released segments)")
        return rep.arena.reserve(total)

    def _segment(self, query_id, key, replica, total) -> IndexSegment:
        seg = self.segments.get((query_id, key, replica))
        if seg is None:
            first = self._reserve(self.replicas[replica], total)
            seg = IndexSegment(replica, first, first + total)
            self.segments[(query_id, key, replica)] = seg
        return seg

    def _local_segment(self, query_id, key, replica) -> IndexSegment:
        """The query's index on `replica`; copied from its home GPU over NVLink on first use."""
        seg = self.segments.get((query_id, key, replica))
        if seg is not None:
            return seg
        home = self.segments.get((query_id, key, self.home(query_id)))
        if home is None:
            raise CapacityExceeded(f"index {key!r} of {query_id} was never ingested")
        n = home.row_end - home.row_beg
        src = self.replicas[home.replica]
        dst_rep = self.replicas[replica]
        first = self._reserve(dst_rep, n)
        ingested = torch.cuda.Event()
        ingested.record(src.stream)
        # peer copy over NVLink, ordered after the ingest by an event (torch issues a
        # cross-device copy on the source device's current stream, then orders the
        # destination's current stream, the replica stream here, after it)
        torch.cuda.current_stream(src.device).wait_event(ingested)
        with self._on(dst_rep):
            dst_rep.arena.data()[first:first + n].copy_(
                src.arena.data()[home.row_beg:home.row_end], non_blocking=True)
        seg = IndexSegment(replica, first, first + n, n)
        self.segments[(query_id, key, replica)] = seg
        return seg

    # -- execution ------------------------------------------------------------------------
    def launch(self, profile: EngineProfile, plan, instance):
        """Enqueue the batch's kernels on the replica stream without waiting; returns the
        (start, end) CUDA events bracketing them."""
        if not plan.entries:
            raise CapacityExceeded("empty batch")
        rep = self.replica_for(instance)
        self._waited = {}
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        with self._on(rep):
            # inputs are assembled first; `start` is recorded right before the library calls,
            # so the measured window is the device work of the batch
            # `end` is recorded by the batch right after its library calls and doubles as the
            # results' ready event (one event record fewer per batch)
            if profile.category == "search":
                rec = self._search_batch(rep, plan, start, end)
            else:
                rec = self._rerank_batch(rep, plan, start, end)
        self.launches += 1
        rec.engine_id, rec.replica, rec.start, rec.end = (profile.engine_id,
                                                          self.replicas.index(rep), start, end)
        self.records.append(rec)
        return start, end

    def launch_chain(self, profile: EngineProfile, plan, instance, reranks):
        """One launch for a batch of Searching requests AND the Reranking node each feeds
        (StreamRuntime's fused chain dispatch): every entry searches its own per-query index
        segment (<= 1024 rows) with its query vector, keeps the node's top-k, and reranks those
        hits against the query's question, keeping the rerank node's top_k — the segment
        kernel (tsv_search_rerank_segmented). Both nodes' results go to their accumulators.
        Returns (start, end) events, or None when the batch does not fit the kernel (the
        caller then launches the search alone)."""
        rep = self.replica_for(instance)
        if rep.arena.storage not in ("bf16", "bf16_tiled") or self.dim > 2048:
            return None
        self._waited = {}
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        with self._on(rep):
            qs, qr, rows, meta = [], [], [], []
            k_s = k_r = 1
            for (task, n), rr in zip(plan.entries, reranks):
                node = task.node
                key_out = next(iter(node.meta.outputs))
                k = node.meta.outputs[key_out].items
                top_k = rr.meta.outputs[next(iter(rr.meta.outputs))].items
                idx = self._inputs(task.ctx, node, "index")
                seg = self._local_segment(task.ctx.query_id, idx[0][1][1], self.replicas.index(rep))
                if seg.row_end - seg.row_beg > 1024 or top_k > k:
                    return None
                qs.append(self._query_rows(rep, task, 0, 1))
                qr.append(self._question(rep, task.ctx).reshape(1, -1))
                rows += [seg.row_beg, seg.row_end]
                meta.append((task, rr, k, top_k))
                k_s, k_r = max(k_s, k), max(k_r, top_k)
            q = torch.cat(qs) if len(qs) > 1 else qs[0]
            qq = torch.cat(qr) if len(qr) > 1 else qr[0]
            if qq.dtype != q.dtype:
                qq = qq.to(q.dtype)
            # the segment table goes to the library as a host list (its pinned staging slots)
            max_rows = max(b - a for a, b in zip(rows[::2], rows[1::2]))
            start.record(rep.stream)
            (ss, si), (rs, ri) = rep.arena.search_rerank_segmented(
                q, rows, max(1, max_rows), k_s, k_r, q_rerank=qq, local_ids=True,
                stream=rep.stream)
            end.record(rep.stream)
            ready = end
        r = self.replicas.index(rep)
        for j, (task, rr, k, top_k) in enumerate(meta):
            self.acc.setdefault((task.ctx.query_id, task.node_id), []).append(
                (0, ss[j:j + 1, :k], si[j:j + 1, :k], ready, r))
            self.acc.setdefault((task.ctx.query_id, rr.node_id), []).append(
                (0, rs[j:j + 1, :top_k], ri[j:j + 1, :top_k], ready, r))
        self.launches += 1
        rows_n = sum(b - a for a, b in zip(rows[::2], rows[1::2]))
        rec = LaunchRecord(profile.engine_id, r, "search+rerank", len(meta), rows_n, k_s, self.dim,
                           bytes=rows_n * self.dim * 2 + len(meta) * self.dim * 4 +
                           len(meta) * (k_s + k_r) * 8,
                           flops=4 * rows_n * self.dim, start=start, end=end)
        self.records.append(rec)
        return start, end

    def execute(self, profile: EngineProfile, plan, t: float, instance) -> tuple[float, float | None]:
        """Simulator hook: run the batch; duration = profile latency ("profile") or the device
        time of the launches ("measured", synchronises on the batch's end event)."""
        start, end = self.launch(profile, plan, instance)
        if self.timing == TIMING_MEASURED:
            end.synchronize()
            ms = start.elapsed_time(end)
            self.device_ms_total += ms
            return ms, ms
        return latency(profile, plan.load), None

    def _in_edges(self, graph) -> dict:
        """node id -> [(producer, key)] of its keyed input edges, built once per graph (a batch
        looks its inputs up several times; scanning every edge each time cost more host time
        than the lookups)."""
        got = self._edge_index.get(id(graph))
        if got is None or got[0] is not graph or got[1] != len(graph.edges):
            idx: dict = {}
            for e in graph.edges:
                if e.key is not None:
                    idx.setdefault(e.dst, []).append((e.src, e.key))
            got = (graph, len(graph.edges), idx)
            self._edge_index[id(graph)] = got
        return got[2]

    def _wait(self, rep: Replica, ev) -> None:
        """rep.stream waits for `ev` once per launch: a batch's entries often share producer
        events (one query's results, one upstream batch), and every cudaStreamWaitEvent is a
        few microseconds of host time."""
        key = (id(rep), id(ev))
        if key not in self._waited:
            self._waited[key] = ev  # (holds the event: its id stays unique during the launch)
            rep.stream.wait_event(ev)

    def _inputs(self, ctx, node, want: str):
        """Data arriving on the node's input edges whose producer tag is `want`."""
        out = []
        for src, key in self._in_edges(ctx.graph).get(node.node_id, ()):
            d = ctx.data.get((src, key))
            if isinstance(d, tuple) and d[0] == want:
                out.append((src, d))
            elif want == "result" and isinstance(d, SearchResult):
                out.append((src, d))
        return out

    def _query_rows(self, rep, task, lo: int, hi: int) -> torch.Tensor:
        """Query vectors for requests [lo, hi) of a Searching task (node-relative), assembled
        from the embedding producers' slices."""
        ctx, node = task.ctx, task.node
        key_out = next(iter(node.meta.outputs))
        q_lo_node, _ = _stage_queries(node, key_out)
        a, b = q_lo_node + lo, q_lo_node + hi
        parts = []
        for _, d in sorted(self._inputs(ctx, node, "queries"), key=lambda x: x[1][2]):
            _, key, s_lo, s_hi, total, vecs, ready = d
            x0, x1 = max(a, s_lo), min(b, s_hi)
            if x0 < x1:
                self._wait(rep, ready)
                parts.append(vecs[x0 - s_lo:x1 - s_lo].to(rep.device))
        if not parts or sum(p_.shape[0] for p_ in parts) != b - a:
            raise CapacityExceeded(f"{node.node_id}: query vectors for [{a}, {b}) not available")
        return torch.cat(parts) if len(parts) > 1 else parts[0]

    def _search_batch(self, rep: Replica, plan, start: torch.cuda.Event,
                      end: torch.cuda.Event) -> LaunchRecord:
        """One topology-aware batch of Searching requests: entries with a per-query index input
        become one segmented launch (each entry searches its own query's segment); entries
        without one search the resident global corpus in one launch. A batch mixing both runs
        the two launches back to back on the replica stream."""
        seg_q, seg_off, seg_ranges, seg_meta = [], [0], [], []
        glob_q, glob_meta = [], []
        kmax = 1
        for task, n in plan.entries:
            node = task.node
            key_out = next(iter(node.meta.outputs))
            k = node.meta.outputs[key_out].items // max(1, node.meta.batch_items)
            kmax = max(kmax, k)
            lo = task.next_request
            rows = self._query_rows(rep, task, lo, lo + n)
            idx = self._inputs(task.ctx, node, "index")
            if idx:
                seg = self._local_segment(task.ctx.query_id, idx[0][1][1],
                                          self.replicas.index(rep))
                seg_q.append(rows)
                seg_off.append(seg_off[-1] + n)
                seg_ranges.append((seg.row_beg, seg.row_end))
                seg_meta.append((task, lo, n, k))
            else:
                if self.global_index is None:
                    raise CapacityExceeded(f"{node.node_id}: no index input and no global corpus")
                glob_q.append(rows)
                glob_meta.append((task, lo, n, k))
        if kmax > 128:
            raise ConfigParse(f"per_query_top_k={kmax} exceeds the fused kernel's limit (128)")
        q_seg = (torch.cat(seg_q) if len(seg_q) > 1 else seg_q[0]) if seg_q else None
        q_glob = (torch.cat(glob_q) if len(glob_q) > 1 else glob_q[0]) if glob_q else None
        if q_glob is not None and self.global_index.device != rep.device:
            raise ConfigParse(f"the global corpus is searched from {self.global_index.device}; "
                              f"bind the search engine's replicas there (got {rep.device})")
        start.record(rep.stream)
        launches = []
        if q_seg is not None:
            out = rep.arena.search_segmented(q_seg, seg_off, seg_ranges, kmax, local_ids=True,
                                             stream=rep.stream)
            launches.append((out, seg_meta))
        if q_glob is not None:
            out = self.global_index.search(q_glob, kmax, stream=rep.stream)
            launches.append((out, glob_meta))
        end.record(rep.stream)
        ready = end
        r = self.replicas.index(rep)
        for (scores, ids), metas in launches:
            a = 0
            for task, lo, n, k in metas:
                self.acc.setdefault((task.ctx.query_id, task.node_id), []).append(
                    (lo, scores[a:a + n, :k], ids[a:a + n, :k], ready, r))
                a += n
        nq = sum(n for _, _, n, _ in seg_meta + glob_meta)
        g_rows = self.global_index.rows if glob_meta else 0
        rows = sum(b - a for a, b in seg_ranges) + g_rows
        pairs = (sum((seg_off[i + 1] - seg_off[i]) * (b - a) for i, (a, b) in enumerate(seg_ranges))
                 + sum(n for _, _, n, _ in glob_meta) * g_rows)
        return LaunchRecord("", 0, "search", nq, rows, kmax, self.dim,
                            bytes=rows * self.dim * 2 + nq * self.dim * 2 + nq * kmax * 8,
                            flops=2 * pairs * self.dim)

    def _question(self, rep: Replica, ctx) -> torch.Tensor:
        got = ctx.data.get(("__question__", None))
        if got is None:  # (graphs submitted without on_submit)
            with self._on(rep):
                qv = self.data.question(rep.device, ctx.query_id)
            return qv
        qv, ready = got
        self._wait(rep, ready)
        return qv if qv.device == rep.device else qv.to(rep.device)

    def _rerank_batch(self, rep: Replica, plan, start: torch.cuda.Event,
                      end: torch.cuda.Event) -> LaunchRecord:
        """One batch of Reranking requests = ONE K3 launch: question j scores its own candidate
        row (ids local to its query's index segment, offset on the device by the segment's
        first arena row), duplicates dropped, the best max(top_k) kept; each entry takes its
        top_k. Inputs are assembled before `start`; nothing but the launch sits inside the
        measured window."""
        jobs = []
        for task, n in plan.entries:
            node, ctx = task.node, task.ctx
            key_out = next(iter(node.meta.outputs))
            top_k = node.meta.outputs[key_out].items
            cands = self._inputs(ctx, node, "result")
            if not cands:
                raise CapacityExceeded(f"{node.node_id}: no candidate input")
            res = cands[0][1]
            if res.ready is not None:
                self._wait(rep, res.ready)
            lo = task.next_request
            part = res.ids.reshape(-1)[lo:lo + n]
            idx = self._inputs(ctx, node, "index") or self._index_of_search(ctx, cands[0][0])
            seg = self._local_segment(ctx.query_id, idx[0][1][1], self.replicas.index(rep))
            jobs.append((task, lo, top_k, seg, self._question(rep, ctx), part))
        n_c = max(j[5].shape[0] for j in jobs)
        k_out = max(j[2] for j in jobs)
        if len(jobs) == 1:
            cand = jobs[0][5].reshape(1, -1)
            qs = jobs[0][4].reshape(1, -1)
        else:
            with self._on(rep):
                if all(j[5].shape[0] == n_c for j in jobs):
                    cand = torch.stack([j[5] for j in jobs])
                else:  # pad short candidate rows with -1 (K3 skips them)
                    cand = torch.stack([torch.nn.functional.pad(j[5], (0, n_c - j[5].shape[0]),
                                                                value=-1) for j in jobs])
                qs = torch.cat([j[4].reshape(1, -1) for j in jobs])
        # segment offsets go to the library as a host list (uploaded through its pinned slots)
        offs = [j[3].row_beg for j in jobs]
        if not cand.is_contiguous():
            cand = cand.contiguous()
        start.record(rep.stream)
        s_all, i_all = rep.arena.rerank(qs, cand, k_out, stream=rep.stream, row_offsets=offs)
        end.record(rep.stream)
        ready = end
        r = self.replicas.index(rep)
        for j, (task, lo, top_k, seg, qv, part) in enumerate(jobs):
            self.acc.setdefault((task.ctx.query_id, task.node_id), []).append(
                (lo, s_all[j:j + 1, :top_k], i_all[j:j + 1, :top_k], ready, r))
        n_rows = sum(j[5].shape[0] for j in jobs)
        return LaunchRecord("", 0, "rerank", len(jobs), n_rows, k_out, self.dim,
                            bytes=n_rows * (self.dim * 2 + 4) + len(jobs) * (self.dim * 2 + k_out * 8),
                            flops=2 * n_rows * self.dim)

    def _index_of_search(self, ctx, producer: str):
        """Walk back from an Aggregate / Searching producer to the Searching node's index input."""
        seen = {producer}
        frontier = [producer]
        while frontier:
            nid = frontier.pop()
            node = ctx.graph.nodes[nid]
            if node.kind is PrimitiveKind.SEARCHING:
                got = self._inputs(ctx, node, "index")
                if got:
                    return got
            for e in ctx.graph.edges:
                if e.dst == nid and e.src not in seen:
                    seen.add(e.src)
                    frontier.append(e.src)
        raise CapacityExceeded("rerank candidates do not trace back to an indexed search")

    def _finalize(self, ctx, node) -> None:
        """All requests of a retrieval node are done: assemble its output from the per-batch
        partial results (batches may have split the node's requests)."""
        parts = self.acc.pop((ctx.query_id, node.node_id), [])
        if not parts:
            return
        parts.sort(key=lambda p: p[0])
        key = next(iter(node.meta.outputs))
        rep = self.replicas[parts[0][4]]
        with self._on(rep):
            for ev in {id(p_[3]): p_[3] for p_ in parts}.values():
                rep.stream.wait_event(ev)
            if node.kind is PrimitiveKind.SEARCHING:
                q_lo, q_hi = _stage_queries(node, key)
                res = SearchResult(torch.cat([p_[1] for p_ in parts]),
                                   torch.cat([p_[2] for p_ in parts]), q_lo, q_hi,
                                   node.meta.slice_of.get(key), replica=parts[0][4])
            else:
                top_k = node.meta.outputs[key].items
                if len(parts) == 1:
                    s_, i_ = parts[0][1], parts[0][2]
                else:  # candidates split across batches: merge the partial top-k lists (K4)
                    s_, i_ = merge_topk(torch.stack([p_[1] for p_ in parts]),
                                        torch.stack([p_[2] for p_ in parts]), top_k,
                                        stream=rep.stream, dedup=True)
                res = SearchResult(s_, i_, 0, 1, None, replica=parts[0][4])
            res.ready = self._record(rep)
        ctx.data[(node.node_id, key)] = res

    def finish(self) -> None:
        for rep in self.replicas:
            rep.stream.synchronize()


_GET_STREAM = getattr(torch._C, "_cuda_getCurrentStream", None)
_SET_STREAM = getattr(torch._C, "_cuda_setStream", None)


class _StreamCtx:
    """Make the replica's device and stream current for torch ops issued inside (and restore
    both on exit). Uses torch's raw stream accessors when present: torch.cuda.device +
    torch.cuda.stream build Stream objects on every entry (~10-20 us per use, several uses per
    retrieval batch on the runtime's critical path)."""

    def __init__(self, rep: Replica):
        self.rep = rep

    def __enter__(self):
        rep = self.rep
        idx = rep.device.index
        if _GET_STREAM is None or _SET_STREAM is None:
            self._slow = (torch.cuda.device(rep.device), torch.cuda.stream(rep.stream))
            for c in self._slow:
                c.__enter__()
            return rep
        self._slow = None
        self._prev_dev = torch.cuda.current_device()
        if self._prev_dev != idx:
            torch.cuda.set_device(idx)
        self._prev = _GET_STREAM(idx)  # (stream id, device index, device type)
        st = rep.stream
        _SET_STREAM(stream_id=st.stream_id, device_index=st.device_index,
                    device_type=st.device_type)
        return rep

    def __exit__(self, *exc):
        if self._slow is not None:
            for c in reversed(self._slow):
                c.__exit__(*exc)
            return False
        sid, didx, dtype = self._prev
        _SET_STREAM(stream_id=sid, device_index=didx, device_type=dtype)
        if self._prev_dev != self.rep.device.index:
            torch.cuda.set_device(self._prev_dev)
        return False


def _stage_queries(node: PrimitiveNode, key: str) -> tuple[int, int]:
    out = node.meta.outputs[key]
    s = node.meta.slice_of.get(key)
    if s is None:
        return 0, node.meta.batch_items
    k = out.items // max(1, node.meta.batch_items)
    return s[0] // k, s[1] // k
