"""Instance exchange: the `rlx-instance/1` JSON format and the adapter that
accepts the reference's own `rlmux` objects.

`rlx-instance/1` carries exactly what the scheduling path reads: per
pipeline the latency model, the migration-cost fields of the spec, and the
nodes/edges of its Sub-Stage Graph; plus the instance knobs and the
slowdown table (or "default"). The reference's `save_graph` cannot be used
because it drops `spec` (rlmux/graph.py:451-480).

`as_instance(x)` takes either this package's `Instance` or an `rlmux`
`Instance` (duck-typed via kind `.value` strings) so that
`lookahead_schedule` is a drop-in for callers of the reference.
"""

from __future__ import annotations

import gzip
import json

from .model import (
    Exclusive,
    Instance,
    Merge,
    Multiplex,
    PipelineSpec,
    ResourceAllocation,
    SlowdownModel,
    SlowdownTable,
    SubStage,
    SubStageGraph,
    SubStageKind,
    default_table,
)

FORMAT = "rlx-instance/1"


def _kind(v) -> SubStageKind:
    return SubStageKind(v if isinstance(v, str) else v.value)


def table_from_json(rows) -> SlowdownTable:
    if rows == "default":
        return default_table()
    entries = {}
    for kind, partner, alpha, memv, factor in rows:
        entries[(_kind(kind), None if partner == "-" else _kind(partner), float(alpha), float(memv))] = float(factor)
    return SlowdownTable(entries)


def instance_from_json(d: dict) -> Instance:
    if d.get("format") != FORMAT:
        raise ValueError(f"not an {FORMAT} document")
    graphs = []
    for gd in d["graphs"]:
        pid = gd["pipeline_id"]
        nodes = {}
        ids = []
        for row in gd["nodes"]:
            nid, worker, kind, dur, mem, rem, act, ctx, tok, s0, s1 = row
            nodes[nid] = SubStage(id=nid, pipeline_id=pid, worker_id=int(worker), kind=_kind(kind),
                                  duration=float(dur), mem_fraction=float(mem), step_span=(int(s0), int(s1)),
                                  remaining_decode_tokens=int(rem), active_requests=int(act),
                                  context_tokens=int(ctx), token_total=int(tok))
            ids.append(nid)
        edges = {(ids[s], ids[t]) for s, t in gd["edges"]}
        spec = None
        if gd.get("spec") is not None:
            s = gd["spec"]
            spec = PipelineSpec(pid, float(s["model_params"]), float(s["device_peak_flops"]), float(s["prefill_mfu"]))
        latency = {int(k): float(v) for k, v in gd["latency"]}
        graphs.append(SubStageGraph(pid, nodes, edges, spec, latency))
    return Instance(graphs=graphs, model=SlowdownModel(table_from_json(d["table"])),
                    headroom=float(d["headroom"]), realloc_penalty=float(d["realloc_penalty"]),
                    default_migration_cost=float(d["default_migration_cost"]),
                    merge_enabled=bool(d["merge_enabled"]))


def instance_to_json(inst: Instance) -> dict:
    rows = []
    for (kind, partner, alpha, memv), f in inst.model.table.entries.items():
        rows.append([kind.value, partner.value if partner else "-", alpha, memv, f])
    rows.sort(key=lambda r: (r[0], "" if r[1] == "-" else r[1], r[2], r[3]))
    graphs = []
    for g in inst.graphs:
        ids = list(g.nodes)
        idx = {nid: i for i, nid in enumerate(ids)}
        nodes = [[n.id, n.worker_id, n.kind.value, n.duration, n.mem_fraction, n.remaining_decode_tokens,
                  n.active_requests, n.context_tokens, n.token_total, n.step_span[0], n.step_span[1]]
                 for n in (g.nodes[i] for i in ids)]
        spec = None if g.spec is None else {"model_params": g.spec.model_params,
                                             "device_peak_flops": g.spec.device_peak_flops,
                                             "prefill_mfu": g.spec.prefill_mfu}
        graphs.append({"pipeline_id": g.pipeline_id, "latency": sorted([int(k), v] for k, v in g.latency_model.items()),
                       "spec": spec, "nodes": nodes, "edges": sorted([idx[s], idx[t]] for s, t in g.edges)})
    return {"format": FORMAT, "headroom": inst.headroom, "realloc_penalty": inst.realloc_penalty,
            "default_migration_cost": inst.default_migration_cost, "merge_enabled": inst.merge_enabled,
            "table": rows, "graphs": graphs}


def load_instance(path: str) -> Instance:
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        return instance_from_json(json.load(fh))


def load_instances(path: str) -> dict:
    """A gz/JSON dict of name -> rlx-instance/1 documents."""
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        blob = json.load(fh)
    return {k: instance_from_json(v) for k, v in blob.items()}


def save_instance(inst: Instance, path: str) -> None:
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "wt", encoding="utf-8") as fh:
        json.dump(instance_to_json(inst), fh, separators=(",", ":"))


# ---------------------------------------------------------------------------
# Reference interop


def is_reference_instance(x) -> bool:
    return type(x).__module__.startswith("rlmux")


def as_instance(x) -> Instance:
    """This package's Instance, converting an rlmux Instance if needed."""
    if isinstance(x, Instance):
        return x
    if not hasattr(x, "graphs") or not hasattr(x, "model"):
        raise TypeError(f"expected an Instance, got {type(x).__name__}")
    graphs = []
    for g in x.graphs:
        nodes = {}
        for nid, n in g.nodes.items():
            nodes[nid] = SubStage(id=n.id, pipeline_id=n.pipeline_id, worker_id=n.worker_id, kind=_kind(n.kind),
                                  duration=n.duration, mem_fraction=n.mem_fraction, step_span=tuple(n.step_span),
                                  sample_ids=frozenset(n.sample_ids),
                                  remaining_decode_tokens=n.remaining_decode_tokens,
                                  active_requests=n.active_requests, context_tokens=n.context_tokens,
                                  token_total=n.token_total)
        spec = None
        if g.spec is not None:
            spec = PipelineSpec(g.pipeline_id, g.spec.model_params, g.spec.device_peak_flops, g.spec.prefill_mfu)
        graphs.append(SubStageGraph(g.pipeline_id, nodes, set(g.edges), spec, dict(g.latency_model)))
    entries = {}
    for (k, p, a, m), f in x.model.table.entries.items():
        entries[(_kind(k), None if p is None else _kind(p), a, m)] = f
    return Instance(graphs=graphs, model=SlowdownModel(SlowdownTable(entries)), headroom=x.headroom,
                    realloc_penalty=x.realloc_penalty, default_migration_cost=x.default_migration_cost,
                    merge_enabled=x.merge_enabled)


def action_as(action, like_module):
    """Re-express one of our actions with the classes of `like_module`
    (e.g. rlmux.scheduler) so callers can hand the schedule back to the
    reference's `simulate`."""
    RA = like_module.ResourceAllocation
    if isinstance(action, Exclusive):
        return like_module.Exclusive(action.node_id, RA(action.alloc.sm_share, action.alloc.mem_share))
    if isinstance(action, Multiplex):
        return like_module.Multiplex(action.node_a, action.node_b, RA(action.alloc_a.sm_share, action.alloc_a.mem_share))
    return like_module.Merge(tuple(action.member_ids), action.target_worker)


def action_from(action):
    """Inverse of `action_as`: accept a reference (or our) action."""
    name = type(action).__name__
    if name == "Exclusive":
        return Exclusive(action.node_id, ResourceAllocation(action.alloc.sm_share, action.alloc.mem_share))
    if name == "Multiplex":
        return Multiplex(action.node_a, action.node_b,
                         ResourceAllocation(action.alloc_a.sm_share, action.alloc_a.mem_share))
    if name == "Merge":
        return Merge(tuple(action.member_ids), action.target_worker)
    raise TypeError(f"unknown action {action!r}")


def action_to_json(a) -> list:
    if isinstance(a, Exclusive):
        return ["X", a.node_id, a.alloc.sm_share, a.alloc.mem_share]
    if isinstance(a, Multiplex):
        return ["M", a.node_a, a.node_b, a.alloc_a.sm_share, a.alloc_a.mem_share]
    return ["G", list(a.member_ids), a.target_worker]


def action_from_json(j):
    if j[0] == "X":
        return Exclusive(j[1], ResourceAllocation(j[2], j[3]))
    if j[0] == "M":
        return Multiplex(j[1], j[2], ResourceAllocation(j[3], j[4]))
    return Merge(tuple(j[1]), int(j[2]))


def to_reference(inst: Instance):
    """This package's Instance -> the reference's own objects (the inverse of
    `as_instance`; needs an importable `rlmux`). Pipeline specs become
    records of the fields the scheduling path reads (migration_cost,
    rlmux/scheduler.py:174-182); the generator-only PipelineSpec fields
    (stages, samples) are not part of an Instance's scheduling semantics."""
    import types

    import rlmux.graph as rg
    import rlmux.scheduler as rsch
    import rlmux.slowdown as rsl

    graphs = []
    for g in inst.graphs:
        nodes = {nid: rg.SubStage(id=n.id, pipeline_id=n.pipeline_id, worker_id=n.worker_id,
                                  kind=rg.SubStageKind(n.kind.value), duration=n.duration,
                                  mem_fraction=n.mem_fraction, step_span=tuple(n.step_span),
                                  sample_ids=frozenset(n.sample_ids),
                                  remaining_decode_tokens=n.remaining_decode_tokens,
                                  active_requests=n.active_requests, context_tokens=n.context_tokens,
                                  token_total=n.token_total) for nid, n in g.nodes.items()}
        spec = None if g.spec is None else types.SimpleNamespace(
            pipeline_id=g.pipeline_id, model_params=g.spec.model_params,
            device_peak_flops=g.spec.device_peak_flops, prefill_mfu=g.spec.prefill_mfu)
        graphs.append(rg.SubStageGraph(g.pipeline_id, nodes, set(g.edges), spec, dict(g.latency_model)))
    entries = {(rg.SubStageKind(k.value), None if p is None else rg.SubStageKind(p.value), a, m): f
               for (k, p, a, m), f in inst.model.table.entries.items()}
    return rsch.Instance(graphs=graphs, model=rsl.SlowdownModel(rsl.SlowdownTable(entries)),
                         headroom=inst.headroom, realloc_penalty=inst.realloc_penalty,
                         default_migration_cost=inst.default_migration_cost, merge_enabled=inst.merge_enabled)
