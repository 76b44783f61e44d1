"""Reference-side harness (TEST INFRASTRUCTURE ONLY — runs in the build
container, never on the GPU box and never on the product path).

It imports the upstream `rlmux` package from /root/reference/pkg/src and
turns it into golden data for this repo:

* the five BASELINE.json config instances, built with the reference's own
  generator (`workload.generate_synthetic` -> `expand_to_trace` ->
  `graph.construct_graph`), plus the trap and random fixtures;
* an instrumented look-ahead chooser that records, per decision, the
  candidate count and the winning key (cost, finish, priority, serial)
  exactly as `scheduler.py:963-972` builds it;
* per-candidate (cost, finish) keys for sampled candidates.

Instances are serialised to the repo's own JSON format (`rlx-instance/1`,
read by `paper_2604_23838_b200.instance_io`), because `save_graph`
drops `spec` (graph.py:451-480) and pickles would need rlmux to load.
"""

from __future__ import annotations

import gzip
import itertools
import json
import os
import sys

REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import rlmux.scheduler as rs  # noqa: E402
from rlmux import fixtures as rf  # noqa: E402
from rlmux.graph import MERGEABLE_KINDS, SubStage, SubStageGraph, SubStageKind, construct_graph  # noqa: E402
from rlmux.scheduler import (  # noqa: E402
    Candidate,
    Exclusive,
    ExecState,
    Instance,
    Merge,
    Multiplex,
    _drive,
    action_finish_estimate,
    candidate_cost,
    feasible,
)
from rlmux.slowdown import MEM_GRID, ResourceAllocation, default_model  # noqa: E402
from rlmux.workload import GeneratorConfig, expand_to_trace, generate_synthetic  # noqa: E402

_ORIG_ENUMERATE = rs.enumerate_actions


# ---------------------------------------------------------------------------
# Capped enumerator (same order and serial semantics as scheduler.py:648-703,
# with merge-set sizes limited to max_merge). max_merge=None == reference.


def capped_enumerate(state: ExecState, max_merge: int | None = None) -> list[Candidate]:
    instance = state.instance
    idle = set(state.idle_workers())
    ready = state.ready_compute()
    out: list[Candidate] = []
    serial = 0
    by_worker: dict[int, list[SubStage]] = {}
    for node in ready:
        by_worker.setdefault(node.worker_id, []).append(node)
    for worker in sorted(by_worker):
        if worker not in idle:
            continue
        for a, b in itertools.combinations(by_worker[worker], 2):
            if a.pipeline_id == b.pipeline_id:
                continue
            if not feasible(a.mem_fraction, b.mem_fraction, instance.headroom):
                continue
            for first, second in ((a, b), (b, a)):
                for alpha in rs.MUX_SM_GRID:
                    for memv in MEM_GRID:
                        if memv + second.mem_fraction > 1.0 - instance.headroom + rs._EPS:
                            continue
                        out.append(Candidate(serial, 0, Multiplex(first.id, second.id, ResourceAllocation(alpha, memv))))
                        serial += 1
    by_pipe: dict[str, list[SubStage]] = {}
    if instance.merge_enabled:
        for node in ready:
            if node.kind in MERGEABLE_KINDS:
                by_pipe.setdefault(node.pipeline_id, []).append(node)
    for pid in sorted(by_pipe):
        frags = by_pipe[pid]
        if len(frags) < 2:
            continue
        top = len(frags) if max_merge is None else min(len(frags), max_merge)
        for size in range(2, top + 1):
            for combo in itertools.combinations(frags, size):
                workers = [m.worker_id for m in combo]
                if len(set(workers)) != len(workers):
                    continue
                ids = tuple(sorted(m.id for m in combo))
                for target in sorted(workers):
                    out.append(Candidate(serial, 1, Merge(ids, target)))
                    serial += 1
    for node in ready:
        if node.worker_id in idle:
            out.append(Candidate(serial, 2, Exclusive(node.id)))
            serial += 1
    return out


class capped:
    """Context manager installing the capped enumerator into rlmux.scheduler
    (module-global lookup at scheduler.py:939 and :912)."""

    def __init__(self, max_merge):
        self.max_merge = max_merge

    def __enter__(self):
        mm = self.max_merge
        rs.enumerate_actions = lambda st: capped_enumerate(st, mm)
        return self

    def __exit__(self, *exc):
        rs.enumerate_actions = _ORIG_ENUMERATE
        return False


# ---------------------------------------------------------------------------
# Instance builders (BASELINE.md §3 / SURVEY.md §8(d) recipes)


def _pipeline(pid, params, seed, batch, workers, sigma=1.0, **kw):
    cfg = GeneratorConfig(batch=batch, workers=workers, model_params=params, decode_sigma=sigma,
                          pipeline_id=pid, **kw)
    spec = generate_synthetic(cfg, seed)
    return construct_graph(expand_to_trace(spec), spec=spec)


def _asyncify(g: SubStageGraph) -> SubStageGraph:
    """Config-3 'async' recipe (builder-defined): drop the
    cross-worker Training barrier (graph.py:393-395) keeping only the
    same-worker ref->train edge, and add an independent mid-step Training
    node per worker that is ready at t=0 (fixtures.py:131-138 pattern)."""
    nodes = dict(g.nodes)
    edges = set()
    for src, dst in g.edges:
        d = nodes[dst]
        if d.kind is SubStageKind.TRAINING and nodes[src].worker_id != d.worker_id:
            continue
        edges.add((src, dst))
    lat = g.latency_model
    for w in sorted({n.worker_id for n in g.nodes.values()}):
        sid = f"{g.pipeline_id}/w{w}/mid"
        nodes[sid] = SubStage(id=sid, pipeline_id=g.pipeline_id, worker_id=w, kind=SubStageKind.TRAINING,
                              duration=lat[4], mem_fraction=0.6)
    return SubStageGraph(pipeline_id=g.pipeline_id, nodes=nodes, edges=edges, spec=g.spec,
                         latency_model=dict(lat))


def build_config(k: int) -> Instance:
    if k == 1:
        graphs = [_pipeline("qwen8b", 8e9, 0, 256, 8)]
    elif k == 2:
        graphs = [_pipeline("qwen8b", 8e9, 1, 512, 16), _pipeline("qwen14b", 14e9, 2, 512, 16)]
    elif k == 3:
        graphs = [
            _asyncify(_pipeline(f"p{i}", p, 10 + i, 1024, 32, sigma=1.5))
            for i, p in enumerate((4e9, 8e9, 14e9, 32e9))
        ]
    elif k == 4:
        graphs = [
            _pipeline(f"a{i}", p, 30 + i, 4096, 64, sigma=1.0, tool_prob=0.5, tool_latency_mean=2.0)
            for i, p in enumerate((0.6e9, 4e9, 8e9, 14e9))
        ]
    elif k == 5:
        graphs = [
            _pipeline(f"p{i}", p, 100 + i, 8192, 64, sigma=1.5)
            for i, p in enumerate((4e9, 8e9, 8e9, 14e9, 14e9, 32e9, 4e9, 8e9))
        ]
    else:
        raise ValueError(k)
    return Instance(graphs=graphs, model=default_model())


def build_async_small() -> Instance:
    """2 pipelines x 4 workers version of the config-3 recipe."""
    graphs = [_asyncify(_pipeline(f"p{i}", p, 10 + i, 64, 4, sigma=1.5)) for i, p in enumerate((4e9, 8e9))]
    return Instance(graphs=graphs, model=default_model())


# ---------------------------------------------------------------------------
# Serialisation to rlx-instance/1


def table_to_json(entries) -> list:
    table = []
    for (kind, partner, alpha, memv), factor in sorted(
        entries.items(),
        key=lambda kv: (kv[0][0].value, kv[0][1].value if kv[0][1] else "", kv[0][2], kv[0][3]),
    ):
        table.append([kind.value, partner.value if partner else "-", alpha, memv, factor])
    return table


_DEFAULT_TABLE = None


def instance_to_json(inst: Instance) -> dict:
    global _DEFAULT_TABLE
    if _DEFAULT_TABLE is None:
        _DEFAULT_TABLE = table_to_json(default_model().table.entries)
    table = table_to_json(inst.model.table.entries)
    if table == _DEFAULT_TABLE:
        table = "default"
    graphs = []
    for g in inst.graphs:
        ids = list(g.nodes)
        index = {nid: i for i, nid in enumerate(ids)}
        nodes = []
        for nid in ids:
            n = g.nodes[nid]
            nodes.append([n.id, n.worker_id, n.kind.value, n.duration, n.mem_fraction,
                          n.remaining_decode_tokens, n.active_requests, n.context_tokens,
                          n.token_total, n.step_span[0], n.step_span[1]])
        edges = sorted([index[s], index[d]] for s, d in g.edges)
        spec = None
        if g.spec is not None:
            spec = {"model_params": g.spec.model_params, "device_peak_flops": g.spec.device_peak_flops,
                    "prefill_mfu": g.spec.prefill_mfu}
        graphs.append({"pipeline_id": g.pipeline_id,
                       "latency": sorted([int(k), v] for k, v in g.latency_model.items()),
                       "spec": spec, "nodes": nodes, "edges": edges})
    return {"format": "rlx-instance/1", "headroom": inst.headroom, "realloc_penalty": inst.realloc_penalty,
            "default_migration_cost": inst.default_migration_cost, "merge_enabled": inst.merge_enabled,
            "table": table, "graphs": graphs}


def save_instance_json(inst: Instance, path: str) -> None:
    data = json.dumps(instance_to_json(inst), separators=(",", ":"))
    if path.endswith(".gz"):
        with gzip.open(path, "wt", encoding="utf-8", compresslevel=9) as fh:
            fh.write(data)
    else:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(data)


def action_to_json(a) -> list:
    if isinstance(a, Exclusive):
        return ["X", a.node_id, a.alloc.sm_share, a.alloc.mem_share]
    if isinstance(a, Multiplex):
        return ["M", a.node_a, a.node_b, a.alloc_a.sm_share, a.alloc_a.mem_share]
    return ["G", list(a.member_ids), a.target_worker]


# ---------------------------------------------------------------------------
# Instrumented look-ahead (chooser semantics of scheduler.py:963-972)


def recorded_lookahead(inst: Instance, window: int, max_merge=None, prelude=()):
    decisions = []

    def chooser(state, cands):
        best = None
        best_key = None
        for cand in cands:
            cost = candidate_cost(state, cand.action, window)
            finish = action_finish_estimate(state, cand.action)
            key = (cost, finish, cand.priority, cand.serial)
            if best_key is None or key < best_key:
                best, best_key = cand, key
        decisions.append({"now": state.now, "n": len(cands), "key": list(best_key),
                          "action": action_to_json(best.action)})
        return best

    with capped(max_merge):
        sched = _drive(inst, chooser, "lookahead", {"window": str(window)}, prelude)
    return sched, decisions


def schedule_to_json(sched) -> list:
    return [[t.start, action_to_json(t.action)] for t in sched.actions]


def candidate_keys(state: ExecState, cands, window: int, which=None):
    out = []
    for i in (range(len(cands)) if which is None else which):
        c = cands[i]
        out.append([c.serial, c.priority, candidate_cost(state, c.action, window),
                    action_finish_estimate(state, c.action)])
    return out
