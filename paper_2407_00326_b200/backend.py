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


class RetrievalBackend:
    """Executes batches of the bound retrieval engines on GPU replicas.

    engines: engine ids to serve (default: every engine of category search/rerank that the
    workflow uses for vector search — `vdb-search0`, `rerank0`). `web0` / `tool0` searches
    stay latency-modeled."""

    def __init__(self, dim: int, devices: list[int] | None = None, arena_rows: int = 1 << 20,
                 engines=("vdb-search0", "rerank0"), timing: str = TIMING_PROFILE,
                 data: SyntheticData | None = None, metric: str = "cosine",
                 global_index=None):
        """global_index: the resident corpus searched by Searching nodes that have no per-query
        index input — a DeviceIndex, or a ShardedIndex spanning several devices (shards
        searched concurrently, merged on its root device)."""
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
        pass

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

    def _segment(self, query_id, key, replica, total) -> IndexSegment:
        seg = self.segments.get((query_id, key, replica))
        if seg is None:
            rep = self.replicas[replica]
            with self._on(rep):
                first = rep.arena.append(torch.zeros((total, self.dim), dtype=torch.bfloat16,
                                                     device=rep.device), stream=rep.stream)
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
        src.stream.synchronize()
        with self._on(dst_rep):  # peer copy over NVLink, then append on the local stream
            rows = src.arena.data()[home.row_beg:home.row_end].to(dst_rep.device)
            first = dst_rep.arena.append(rows, stream=dst_rep.stream)
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
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        with self._on(rep):
            # inputs are assembled first; `start` is recorded right before the library calls,
            # so the measured window is the device work of the batch
            if profile.category == "search":
                rec = self._search_batch(rep, plan, start)
            else:
                rec = self._rerank_batch(rep, plan, start)
            end.record(rep.stream)
        self.launches += 1
        rec.engine_id, rec.replica, rec.start, rec.end = (profile.engine_id,
                                                          self.replicas.index(rep), start, end)
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

    def _inputs(self, ctx, node, want: str):
        """Data arriving on the node's input edges whose producer tag is `want`."""
        out = []
        for e in ctx.graph.edges:
            if e.dst == node.node_id and e.key is not None:
                d = ctx.data.get((e.src, e.key))
                if isinstance(d, tuple) and d[0] == want:
                    out.append((e.src, d))
                elif want == "result" and isinstance(d, SearchResult):
                    out.append((e.src, d))
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
                rep.stream.wait_event(ready)
                parts.append(vecs[x0 - s_lo:x1 - s_lo].to(rep.device))
        if not parts or sum(p_.shape[0] for p_ in parts) != b - a:
            raise CapacityExceeded(f"{node.node_id}: query vectors for [{a}, {b}) not available")
        return torch.cat(parts) if len(parts) > 1 else parts[0]

    def _search_batch(self, rep: Replica, plan, start: torch.cuda.Event) -> None:
        qs, q_off, ranges, metas = [], [0], [], []
        kmax = 1
        use_global = False
        for task, n in plan.entries:
            node = task.node
            key_out = next(iter(node.meta.outputs))
            k = node.meta.outputs[key_out].items // max(1, node.meta.batch_items)
            kmax = max(kmax, k)
            lo = task.next_request
            qs.append(self._query_rows(rep, task, lo, lo + n))
            q_off.append(q_off[-1] + n)
            idx = self._inputs(task.ctx, node, "index")
            if idx:
                seg = self._local_segment(task.ctx.query_id, idx[0][1][1],
                                          self.replicas.index(rep))
                ranges.append((seg.row_beg, seg.row_end))
            else:
                if self.global_index is None:
                    raise CapacityExceeded(f"{node.node_id}: no index input and no global corpus")
                use_global = True
                ranges.append((0, self.global_index.rows))
            metas.append((task, lo, n, k))
        q = torch.cat(qs)
        if kmax > 128:
            raise ConfigParse(f"per_query_top_k={kmax} exceeds the fused kernel's limit (128)")
        start.record(rep.stream)
        if use_global:
            if self.global_index.device != rep.device:
                raise ConfigParse(f"the global corpus is searched from {self.global_index.device}; "
                                  f"bind the search engine's replicas there (got {rep.device})")
            scores, ids = self.global_index.search(q, kmax, stream=rep.stream)
        else:
            scores, ids = rep.arena.search_segmented(q, q_off, ranges, kmax, local_ids=True,
                                                     stream=rep.stream)
        ready = self._record(rep)
        r = self.replicas.index(rep)
        for (task, lo, n, k), a in zip(metas, q_off[:-1]):
            self.acc.setdefault((task.ctx.query_id, task.node_id), []).append(
                (lo, scores[a:a + n, :k], ids[a:a + n, :k], ready, r))
        nq = q_off[-1]
        rows = sum(b - a for a, b in ranges)
        pairs = sum((q_off[i + 1] - q_off[i]) * (b - a) for i, (a, b) in enumerate(ranges))
        return LaunchRecord("", 0, "search", nq, rows, kmax, self.dim,
                            bytes=rows * self.dim * 2 + nq * self.dim * 2 + nq * kmax * 8,
                            flops=2 * pairs * self.dim)

    def _rerank_batch(self, rep: Replica, plan, start: torch.cuda.Event) -> None:
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
                rep.stream.wait_event(res.ready)
            flat = res.ids.reshape(-1)
            lo = task.next_request
            part = flat[lo:lo + n]
            idx = self._inputs(ctx, node, "index") or self._index_of_search(ctx, cands[0][0])
            seg = self._local_segment(ctx.query_id, idx[0][1][1], self.replicas.index(rep))
            rows = torch.where(part >= 0, part + seg.row_beg, part).to(torch.int32)
            qv = self.data.question(rep.device, ctx.query_id)
            jobs.append((task, lo, top_k, seg, qv.reshape(1, -1), rows.reshape(-1)))
        # One K3 launch for the whole batch: question j scores its own candidate row (padded
        # with -1, which K3 skips), the best max(top_k) are kept and each job takes its top_k.
        n_c = max(j[5].shape[0] for j in jobs)
        k_out = max(j[2] for j in jobs)
        cand = torch.full((len(jobs), n_c), -1, dtype=torch.int32, device=rep.device)
        for j, job in enumerate(jobs):
            cand[j, :job[5].shape[0]] = job[5]
        qs = torch.cat([j[4] for j in jobs]) if len(jobs) > 1 else jobs[0][4]
        offs = torch.tensor([[j[3].row_beg] for j in jobs], dtype=torch.int32).pin_memory()
        offs = offs.to(rep.device, non_blocking=True)
        start.record(rep.stream)
        s_all, i_all = rep.arena.rerank(qs, cand, k_out, stream=rep.stream)
        i_all = torch.where(i_all >= 0, i_all - offs, i_all)
        ready = self._record(rep)
        r = self.replicas.index(rep)
        for j, (task, lo, top_k, seg, qv, rows) in enumerate(jobs):
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
            for p_ in parts:
                rep.stream.wait_event(p_[3])
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


class _StreamCtx:
    def __init__(self, rep: Replica):
        self.rep = rep
        self._dev = torch.cuda.device(rep.device)
        self._st = torch.cuda.stream(rep.stream)

    def __enter__(self):
        self._dev.__enter__()
        self._st.__enter__()
        return self.rep

    def __exit__(self, *exc):
        self._st.__exit__(*exc)
        self._dev.__exit__(*exc)
        return False


def _stage_queries(node: PrimitiveNode, key: str) -> tuple[int, int]:
    out = node.meta.outputs[key]
    s = node.meta.slice_of.get(key)
    if s is None:
        return 0, node.meta.batch_items
    k = out.items // max(1, node.meta.batch_items)
    return s[0] // k, s[1] // k
