"""Creation and sub-batch splitting of the retrieval primitives (optimizer subset).

Mirrors the parts of pkg/src/teola_sim/optimizer.py that shape the retrieval path:
  * Searching / Reranking node creation (optimizer.py:178-218);
  * the stage machinery shared by Pass 2 and Pass 4: `_even_ranges` (536-537),
    `_even_shares` (540-542), `_splittable_outputs` (545-547), `_split_node` (550-617),
    `_insert_aggregates` (620-661);
  * Pass 2 `stage_decompose` (668-703) — splits a batchable Searching node with more queries
    than the engine's B_eff into ceil(items / B_eff) stages;
  * Pass 4 `pipeline_decode` / `_propagate_split` (782-878) — query-expansion decodes stream
    per segment, and the split propagates into the query-embedding and Searching nodes.
The LLM-only passes (dependency pruning, prefill split) are out of scope.

Every stage carries `slice_of[key] = (start, stop, total)`: the item range of the unsplit
output it produces. The GPU path uses exactly these slices — a Searching stage runs the
queries [start/k, stop/k) and an Aggregate concatenates stage outputs in slice order.
"""

from __future__ import annotations

from .engines import EngineSet, max_efficient_batch
from .errors import ConfigParse
from .graph import (BATCHABLE, CONTROL_KINDS, DECODE_KINDS, PREFILL_KINDS, SPLITTABLE, Edge,
                    MetadataProfile, Payload, PGraph, PrimitiveKind, PrimitiveNode, topo_sort)

CHUNK_TOKENS = 256


class ConfigMissing(ConfigParse):
    def __init__(self, component: str, param: str):
        super().__init__(f"component {component!r} is missing required parameter {param!r}")
        self.component = component
        self.param = param


def _need(name: str, params: dict, key: str):
    if key not in params:
        raise ConfigMissing(name, key)
    return params[key]


def searching_node(name: str, engine: str, params: dict, inputs: tuple[str, ...], out_key: str,
                   annotations: frozenset[str] = frozenset()) -> PrimitiveNode:
    """ROLE_SEARCH decomposition (optimizer.py:178-197): one Searching node over
    `query_count` queries producing query_count x per_query_top_k items (query-major)."""
    queries = int(params.get("query_count", 1))
    top_k = int(_need(name, params, "per_query_top_k"))
    tok = int(params.get("chunk_token_len", CHUNK_TOKENS))
    return PrimitiveNode(f"{name}.search", PrimitiveKind.SEARCHING, MetadataProfile(
        inputs=tuple(inputs), outputs={out_key: Payload(queries * top_k, queries * top_k * tok)},
        engine_id=engine, batch_items=queries, annotations=frozenset(annotations) | {BATCHABLE}))


def reranking_node(name: str, engine: str, params: dict, inputs: tuple[str, ...], out_key: str,
                   annotations: frozenset[str] = frozenset()) -> PrimitiveNode:
    """ROLE_RERANK decomposition (optimizer.py:199-218): candidate_count requests in, top_k
    items out; not batchable unless annotated, so split stages reach it via an Aggregate."""
    cands = int(_need(name, params, "candidate_count"))
    top_k = int(params.get("top_k", 3))
    tok = int(params.get("chunk_token_len", CHUNK_TOKENS))
    return PrimitiveNode(f"{name}.rerank", PrimitiveKind.RERANKING, MetadataProfile(
        inputs=tuple(inputs), outputs={out_key: Payload(top_k, top_k * tok)}, engine_id=engine,
        batch_items=cands, annotations=frozenset(annotations)))


def even_ranges(total: int, size: int) -> list[tuple[int, int]]:
    return [(a, min(a + size, total)) for a in range(0, total, size)]


def even_shares(total: int, parts: int) -> list[int]:
    q, r = divmod(total, parts)
    return [q + (i < r) for i in range(parts)]


def splittable_outputs(node: PrimitiveNode) -> bool:
    b = node.meta.batch_items
    return all(p.items % b == 0 for p in node.meta.outputs.values())


def dedupe(edges: list[Edge]) -> list[Edge]:
    seen: set[Edge] = set()
    out = []
    for e in edges:
        if e.src != e.dst and e not in seen:
            seen.add(e)
            out.append(e)
    return out


def _stage_meta(meta: MetadataProfile, span: int) -> MetadataProfile:
    return MetadataProfile(
        inputs=meta.inputs, outputs={}, engine_id=meta.engine_id, batch_items=span,
        token_counts=dict(meta.token_counts), decode_tokens=meta.decode_tokens,
        context_tokens=meta.context_tokens, out_segments=1, annotations=meta.annotations,
        cached_prefix_tokens=meta.cached_prefix_tokens, query_id=meta.query_id,
        app_id=meta.app_id)


def split_node(g: PGraph, node_id: str, ranges: list[tuple[int, int]]) -> list[str]:
    """Replace a node by per-range stages `<id>.s<i>` and rewire (optimizer.py:550-617).

    Inputs whose producers all carry slices over this node's item total connect
    range-to-range (overlap); every other input is replicated to all stages. Outgoing edges
    are replicated from each stage."""
    node = g.nodes[node_id]
    total = node.meta.batch_items
    stages = []
    for i, (a, b) in enumerate(ranges):
        meta = _stage_meta(node.meta, b - a)
        for key, p in node.meta.outputs.items():
            scale = p.items // total
            prior = node.meta.slice_of.get(key)
            base = prior[0] if prior else 0
            full = prior[2] if prior else p.items
            meta.outputs[key] = Payload((b - a) * scale, round(p.tokens * (b - a) / total))
            meta.slice_of[key] = (base + a * scale, base + b * scale, full)
        sid = f"{node_id}.s{i}"
        g.nodes[sid] = PrimitiveNode(sid, node.kind, meta)
        stages.append(sid)

    incoming: dict[str | None, list[Edge]] = {}
    outgoing = []
    rest = []
    for e in g.edges:
        if e.dst == node_id:
            incoming.setdefault(e.key, []).append(e)
        elif e.src == node_id:
            outgoing.append(e)
        else:
            rest.append(e)
    wired = []
    for key, edges in incoming.items():
        slices = [g.nodes[e.src].meta.slice_of.get(key) if key is not None else None
                  for e in edges]
        aligned = key is not None and all(s is not None and s[2] == total for s in slices)
        if aligned and len(edges) > 1:
            for sid, (a, b) in zip(stages, ranges):
                wired.extend(Edge(e.src, sid, key) for e, (sa, sb, _) in zip(edges, slices)
                             if sa < b and a < sb)
        else:
            wired.extend(Edge(e.src, sid, e.key) for e in edges for sid in stages)
    for e in outgoing:
        wired.extend(Edge(sid, e.dst, e.key) for sid in stages)
    del g.nodes[node_id]
    g.edges = dedupe(rest + wired)
    return stages


def insert_aggregates(g: PGraph) -> bool:
    """One Aggregate per (unsplit non-batchable consumer, key) fed by >= 2 slice-carrying
    producers over a common total; items/tokens are summed (no dedup) (optimizer.py:620-661).
    On the GPU this is the point where stage results are concatenated / merged (K4)."""
    fired = False
    parents = g.parents()
    for cid in list(g.nodes):
        consumer = g.nodes[cid]
        if consumer.kind in CONTROL_KINDS or consumer.batchable:
            continue
        groups: dict[str, list[Edge]] = {}
        for e in parents[cid]:
            if e.key is not None:
                groups.setdefault(e.key, []).append(e)
        for key, edges in groups.items():
            if len(edges) < 2:
                continue
            slices = [g.nodes[e.src].meta.slice_of.get(key) for e in edges]
            if None in slices or len({s[2] for s in slices}) != 1:
                continue
            outs = [g.nodes[e.src].meta.outputs[key] for e in edges]
            agg_id = f"{cid}.agg.{key.replace('/', '_')}"
            g.nodes[agg_id] = PrimitiveNode(agg_id, PrimitiveKind.AGGREGATE, MetadataProfile(
                inputs=(key,), outputs={key: Payload(sum(p.items for p in outs),
                                                     sum(p.tokens for p in outs))},
                query_id=consumer.meta.query_id, app_id=consumer.meta.app_id))
            g.edges = [e for e in g.edges if not (e.dst == cid and e.key == key)]
            g.edges += [Edge(e.src, agg_id, key) for e in edges] + [Edge(agg_id, cid, key)]
            fired = True
    if fired:
        g.edges = dedupe(g.edges)
    return fired


def stage_decompose(g: PGraph, engines: EngineSet | None) -> tuple[PGraph, bool]:
    """Pass 2 (optimizer.py:668-703): micro-batch batchable nodes whose load exceeds B_eff."""
    if engines is None:
        return g, False
    out = g.clone()
    fired = False
    for nid in topo_sort(g):
        node = out.nodes.get(nid)
        if node is None or node.kind in CONTROL_KINDS or not node.batchable:
            continue
        profile = engines.get(node.meta.engine_id)
        if profile is None:
            continue
        beff = max_efficient_batch(profile)
        items = node.meta.batch_items
        if node.kind in PREFILL_KINDS or node.kind in DECODE_KINDS:
            per = (node.meta.prompt_tokens if node.kind in PREFILL_KINDS
                   else max(1, node.meta.context_tokens))
            if items * per <= beff:
                continue
            size = max(1, int(beff // max(1, per)))
        else:
            if items <= beff:
                continue
            size = max(1, int(beff))
        if size >= items or not splittable_outputs(node):
            continue
        split_node(out, nid, even_ranges(items, size))
        fired = True
    if insert_aggregates(out):
        fired = True
    return out, fired


def pipeline_decode(g: PGraph, engines: EngineSet | None = None) -> tuple[PGraph, bool]:
    """Pass 4 (optimizer.py:782-850): a splittable single-item decode with m output segments
    becomes m chained PartialDecoding nodes, and its itemwise batchable consumers split into
    m per-segment stages (e.g. query expansion -> query embedding -> Searching)."""
    out = g.clone()
    fired = False
    for nid in list(out.nodes):
        node = out.nodes.get(nid)
        if node is None or node.kind is not PrimitiveKind.DECODING or not node.splittable:
            continue
        m = node.meta.out_segments
        if m <= 1 or node.meta.batch_items != 1:
            continue
        consumers = [e for e in out.edges if e.src == nid]
        if not consumers:
            continue
        ok = True
        for e in consumers:
            c = out.nodes[e.dst]
            if (not c.batchable or c.kind in CONTROL_KINDS or c.meta.batch_items < m
                    or c.meta.batch_items % m or not splittable_outputs(c)):
                ok = False
        if not ok:
            continue
        shares = even_shares(node.meta.decode_tokens, m)
        chain = f"{nid}.stream"
        pds = []
        for i in range(m):
            meta = MetadataProfile(inputs=node.meta.inputs if i == 0 else (chain,), outputs={},
                                   engine_id=node.meta.engine_id, decode_tokens=shares[i],
                                   context_tokens=node.meta.context_tokens,
                                   query_id=node.meta.query_id, app_id=node.meta.app_id)
            for k, p in node.meta.outputs.items():
                per = p.items // m
                meta.outputs[k] = Payload(per, round(p.tokens / m))
                meta.slice_of[k] = (i * per, (i + 1) * per, p.items)
            if i < m - 1:
                meta.outputs[chain] = Payload(1, node.meta.context_tokens)
            pid = f"{nid}.pd{i}"
            out.nodes[pid] = PrimitiveNode(pid, PrimitiveKind.PARTIAL_DECODING, meta)
            pds.append(pid)
        edges = []
        for e in out.edges:
            if e.dst == nid:
                edges.append(Edge(e.src, pds[0], e.key))
            elif e.src == nid:
                edges.extend(Edge(p, e.dst, e.key) for p in pds)
            else:
                edges.append(e)
        edges += [Edge(pds[i], pds[i + 1], chain) for i in range(m - 1)]
        del out.nodes[nid]
        out.edges = dedupe(edges)
        for e in consumers:
            propagate_split(out, e.dst, m)
        fired = True
    if insert_aggregates(out):
        fired = True
    return out, fired


def propagate_split(g: PGraph, nid: str, parts: int) -> None:
    """Split a consumer into `parts` stages and continue into batchable, itemwise-compatible
    consumers (optimizer.py:853-878)."""
    node = g.nodes.get(nid)
    if node is None or node.meta.slice_of:
        return
    items = node.meta.batch_items
    downstream = list(dict.fromkeys(e.dst for e in g.edges if e.src == nid))
    split_node(g, nid, even_ranges(items, items // parts))
    totals = {k: p.items for k, p in node.meta.outputs.items()}
    for did in downstream:
        child = g.nodes.get(did)
        if child is None or child.meta.slice_of:
            continue
        feeds = {e.key for e in g.edges if e.dst == did and e.key in totals}
        if not feeds:
            continue
        if (child.batchable and child.kind not in CONTROL_KINDS
                and all(totals[k] == child.meta.batch_items for k in feeds)
                and child.meta.batch_items % parts == 0 and splittable_outputs(child)):
            propagate_split(g, did, parts)


def stage_query_range(node: PrimitiveNode, key: str) -> tuple[int, int]:
    """Queries a Searching stage covers: its output slice divided by per-query top-k."""
    out = node.meta.outputs[key]
    s = node.meta.slice_of.get(key)
    if s is None:
        return 0, node.meta.batch_items
    k = out.items // max(1, node.meta.batch_items)
    return s[0] // k, s[1] // k
