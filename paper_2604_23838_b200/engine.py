"""Host execution state for the decision loop.

This is the mutable state the reference's `_drive` loop owns
(rlmux/scheduler.py:339-634, `ExecState`): readiness, action application
(exclusive / multiplex / merge surgery), event advance with survivor
re-rating, and tool-wait auto-start. The look-ahead *scoring* of candidates
never runs here — it runs on the device (`native.py`); this object only
applies the one winning action per decision and advances simulated time,
and it is the source of the per-decision state snapshot the device
consumes (`encode.py`).

Semantics follow the code, not the SPEC:
  * consume(dt): prefix first, then work/rate, clamped at 0 (:330-336)
  * finished iff prefix<=EPS and work*rate<=EPS (:609)
  * survivor of a pair is re-rated to exactly 1.0 / FULL_ALLOCATION (:615-621)
  * tool waits expire at end<=now+EPS, then ready tool waits auto-start (:622-627)
"""

from __future__ import annotations

from dataclasses import dataclass

from .model import (
    DEFAULT_MEM_FRACTIONS,
    EPS,
    FULL_ALLOCATION,
    MERGEABLE_KINDS,
    Exclusive,
    Instance,
    Merge,
    Multiplex,
    ResourceAllocation,
    SchedulingError,
    SubStage,
    SubStageKind,
    complement_allocation,
    feasible,
    merged_estimate,
    migration_cost,
)


@dataclass
class Running:
    node: SubStage
    worker: int
    rate: float
    alloc: ResourceAllocation
    prefix_left: float
    work_left: float
    partner_id: str | None
    started: float

    def finish_estimate(self, now: float) -> float:
        return now + self.prefix_left + self.work_left * self.rate

    def consume(self, dt: float) -> None:
        if self.prefix_left > EPS:
            used = dt if dt < self.prefix_left else self.prefix_left
            self.prefix_left -= used
            dt -= used
        if dt > EPS and self.work_left > EPS:
            rest = self.work_left - dt / self.rate
            self.work_left = rest if rest > 0.0 else 0.0


class HostState:
    """Execution state over an instance's combined sub-stage graphs."""

    def __init__(self, instance: Instance, record: bool = False):
        self.instance = instance
        self.record = record
        self.now = 0.0
        self.makespan = 0.0
        self.nodes: dict[str, SubStage] = {}
        self.preds: dict[str, set] = {}
        self.succs: dict[str, set] = {}
        for g in instance.graphs:
            for nid, node in g.nodes.items():
                self.nodes[nid] = node
                self.preds[nid] = set()
                self.succs[nid] = set()
        for g in instance.graphs:
            for src, dst in g.edges:
                self.preds[dst].add(src)
                self.succs[src].add(dst)
        self.completed: set = set()
        self.completion_time: dict = {}
        self.running: dict[str, Running] = {}
        self.worker_members: dict[int, list] = {w: [] for w in instance.workers()}
        self.toolwaits: dict[str, float] = {}
        self.merge_prefix: dict[str, float] = {}
        self.last_mem_grant: dict = {}
        self.events: list = []
        self.revision = 0  # bumped whenever the node/edge structure changes (merges)
        self._start_ready_toolwaits()

    # -- queries ----------------------------------------------------------

    def done(self) -> bool:
        return len(self.completed) == len(self.nodes)

    def has_events(self) -> bool:
        return bool(self.running) or bool(self.toolwaits)

    def is_ready(self, nid: str) -> bool:
        if nid in self.completed or nid in self.running or nid in self.toolwaits:
            return False
        done = self.completed
        return all(p in done for p in self.preds[nid])

    def ready_compute(self) -> list:
        out = [n for nid, n in self.nodes.items() if n.kind is not SubStageKind.TOOL_WAIT and self.is_ready(nid)]
        out.sort(key=lambda n: (n.pipeline_id, n.id))
        return out

    def idle_workers(self) -> list:
        return sorted(w for w, m in self.worker_members.items() if not m)

    def next_event_time(self):
        times = [m.finish_estimate(self.now) for m in self.running.values()]
        times.extend(self.toolwaits.values())
        return min(times) if times else None

    # -- mutation ---------------------------------------------------------

    def _log(self, worker, kind, nid, alloc="-"):
        if self.record:
            self.events.append((self.now, worker, kind, nid, alloc))

    def _complete(self, nid: str) -> None:
        self.completed.add(nid)
        self.completion_time[nid] = self.now
        if self.now > self.makespan:
            self.makespan = self.now
        self._log(self.nodes[nid].worker_id, "finish", nid)

    def _start_ready_toolwaits(self) -> None:
        again = True
        while again:
            again = False
            for nid in sorted(self.nodes):
                node = self.nodes[nid]
                if node.kind is not SubStageKind.TOOL_WAIT or not self.is_ready(nid):
                    continue
                self._log(node.worker_id, "toolwait-start", nid)
                if node.duration <= EPS:
                    self._complete(nid)
                else:
                    self.toolwaits[nid] = self.now + node.duration
                again = True

    def _check_ready(self, nid: str) -> SubStage:
        if nid not in self.nodes:
            raise SchedulingError(f"unknown sub-stage {nid!r}")
        if not self.is_ready(nid):
            missing = sorted(p for p in self.preds[nid] if p not in self.completed)
            if missing:
                raise SchedulingError(f"dependency violation: {nid} needs edge ({missing[0]}, {nid}) resolved")
            raise SchedulingError(f"sub-stage {nid} is not ready (running or done)")
        node = self.nodes[nid]
        if node.kind is SubStageKind.TOOL_WAIT:
            raise SchedulingError(f"tool wait {nid} is not schedulable")
        return node

    def _start(self, node: SubStage, rate: float, alloc: ResourceAllocation, partner) -> None:
        prefix = self.merge_prefix.pop(node.id, 0.0)
        inst = self.instance
        if node.is_rollout and inst.realloc_penalty > 0:
            key = (node.worker_id, node.pipeline_id)
            last = self.last_mem_grant.get(key)
            if last is not None and abs(last - alloc.mem_share) > EPS:
                prefix += inst.realloc_penalty
            self.last_mem_grant[key] = alloc.mem_share
        self.running[node.id] = Running(node, node.worker_id, rate, alloc, prefix, node.duration, partner, self.now)
        self.worker_members[node.worker_id].append(node.id)
        if prefix > EPS:
            self._log(node.worker_id, "migration", node.id)
        self._log(node.worker_id, "start", node.id, f"{alloc.sm_share:.4f}/{alloc.mem_share:.4f}")

    def apply(self, action) -> None:
        model = self.instance.model
        if isinstance(action, Exclusive):
            node = self._check_ready(action.node_id)
            if self.worker_members[node.worker_id]:
                raise SchedulingError(f"worker {node.worker_id} is busy")
            self._start(node, model.slowdown(node.kind, None, action.alloc), action.alloc, None)
        elif isinstance(action, Multiplex):
            a = self._check_ready(action.node_a)
            b = self._check_ready(action.node_b)
            if a.worker_id != b.worker_id:
                raise SchedulingError("multiplex members must share a worker")
            if a.pipeline_id == b.pipeline_id:
                raise SchedulingError("multiplex members must belong to different pipelines")
            if self.worker_members[a.worker_id]:
                raise SchedulingError(f"worker {a.worker_id} is busy")
            if not feasible(a.mem_fraction, b.mem_fraction, self.instance.headroom):
                raise SchedulingError(f"memory infeasible: {a.id}({a.mem_fraction}) + {b.id}({b.mem_fraction})")
            alloc_b = complement_allocation(action.alloc_a, self.instance.headroom)
            rate_a = model.slowdown(a.kind, b.kind, action.alloc_a)
            rate_b = model.slowdown(b.kind, a.kind, alloc_b)
            self._start(a, rate_a, action.alloc_a, b.id)
            self._start(b, rate_b, alloc_b, a.id)
        elif isinstance(action, Merge):
            self._merge(action)
        else:
            raise SchedulingError(f"unknown action {action!r}")
        self._start_ready_toolwaits()

    def _merge(self, action: Merge) -> None:
        """Graph surgery of rlmux/scheduler.py:517-581."""
        if len(action.member_ids) < 2:
            raise SchedulingError("merge needs at least two fragments")
        members = [self._check_ready(nid) for nid in action.member_ids]
        pid = members[0].pipeline_id
        if any(m.pipeline_id != pid for m in members):
            raise SchedulingError("merge fragments must belong to one pipeline")
        if any(m.kind not in MERGEABLE_KINDS for m in members):
            raise SchedulingError("only small/medium decode fragments can merge")
        workers = [m.worker_id for m in members]
        if len(set(workers)) != len(workers):
            raise SchedulingError("merge fragments must sit on distinct workers")
        if action.target_worker not in workers:
            raise SchedulingError("merge target must hold one of the fragments")
        inst = self.instance
        kind, duration = merged_estimate(members, inst.latency_model_for(pid))
        spec = inst.spec_for(pid)
        prefix = 0.0
        for m in members:
            if m.worker_id == action.target_worker:
                continue
            prefix += migration_cost(m, spec) if spec is not None else inst.default_migration_cost
        mid = "merge[" + "+".join(action.member_ids) + f"]@w{action.target_worker}"
        merged = SubStage(
            id=mid, pipeline_id=pid, worker_id=action.target_worker, kind=kind, duration=duration,
            mem_fraction=max(DEFAULT_MEM_FRACTIONS[kind], max(m.mem_fraction for m in members)),
            step_span=(min(m.step_span[0] for m in members), max(m.step_span[1] for m in members)),
            sample_ids=frozenset().union(*(m.sample_ids for m in members)),
            remaining_decode_tokens=sum(m.remaining_decode_tokens for m in members),
            active_requests=sum(m.active_requests for m in members),
            context_tokens=sum(m.context_tokens for m in members),
            token_total=sum(m.token_total for m in members),
        )
        gone = set(action.member_ids)
        preds = set().union(*(self.preds[m.id] for m in members)) - gone
        succs = set().union(*(self.succs[m.id] for m in members)) - gone
        for m in members:
            for p in self.preds[m.id]:
                self.succs[p].discard(m.id)
            for s in self.succs[m.id]:
                self.preds[s].discard(m.id)
            del self.nodes[m.id], self.preds[m.id], self.succs[m.id]
        self.nodes[mid] = merged
        self.preds[mid] = preds
        self.succs[mid] = succs
        for p in preds:
            self.succs[p].add(mid)
        for s in succs:
            self.preds[s].add(mid)
        self.merge_prefix[mid] = prefix
        self.revision += 1
        self._log(action.target_worker, "merge", mid)

    def advance(self, until: float | None = None) -> None:
        nxt = self.next_event_time()
        if nxt is None:
            if until is None:
                raise SchedulingError("no pending events to advance to")
            self.now = max(self.now, until)
            return
        target = nxt if until is None else min(nxt, until)
        dt = target - self.now
        if not dt > 0.0:
            dt = 0.0
        for m in self.running.values():
            m.consume(dt)
        self.now = target
        finished = sorted(nid for nid, m in self.running.items() if m.prefix_left <= EPS and m.work_left * m.rate <= EPS)
        for nid in finished:
            m = self.running.pop(nid)
            self.worker_members[m.worker].remove(nid)
            self._complete(nid)
            if m.partner_id and m.partner_id in self.running:
                partner = self.running[m.partner_id]
                if partner.rate != 1.0:
                    partner.rate = 1.0
                    partner.alloc = FULL_ALLOCATION
                    self._log(partner.worker, "rerate", partner.node.id, "1.0000/0.8000")
                partner.partner_id = None
        expired = sorted(nid for nid, t in self.toolwaits.items() if t <= self.now + EPS)
        for nid in expired:
            del self.toolwaits[nid]
            self._complete(nid)
        if finished or expired:
            self._start_ready_toolwaits()
