"""Replay of a Schedule into the headline metrics (rlmux/sim.py:118-173).

Used to check the north-star parity clause "fp64 makespan and throughput
estimates agree within 1e-9 relative": the schedule produced by the GPU
chooser is re-executed on the host engine and reduced to makespan,
per-pipeline latency, tokens and aggregate throughput exactly as the
reference's `simulate` does.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .instance_io import action_from, as_instance
from .model import EPS, SchedulingError, SubStageKind


class DependencyViolationError(ValueError):
    """rlmux/sim.py:37"""


@dataclass(frozen=True)
class TimelineEvent:
    """rlmux/sim.py:40-46"""

    time: float
    worker_id: int
    kind: str  # start / finish / rerate / merge / migration / toolwait-start
    node_id: str
    alloc: str = "-"


@dataclass
class SimulationReport:
    """rlmux/sim.py:49-66 (same fields; avg/max step latency are copies of
    the per-pipeline latency there too, :164-165)."""

    makespan: float
    per_pipeline_latency: dict
    per_pipeline_avg_step_latency: dict
    per_pipeline_max_step_latency: dict
    per_pipeline_tokens: dict
    aggregate_throughput: float
    utilization_avg: dict
    utilization_series: dict
    events: list = field(default_factory=list)
    policy: str = ""
    metadata: dict = field(default_factory=dict)

    @property
    def total_tokens(self) -> int:
        return sum(self.per_pipeline_tokens.values())


COMPUTE_BOUND_KINDS = frozenset(
    {SubStageKind.TRAINING, SubStageKind.REFERENCE, SubStageKind.PREFILL_BURST, SubStageKind.DECODE_LARGE})


def utilization(events, makespan: float, workers, kind_of) -> tuple:
    """Per-worker SM-share segments of compute-bound members and their
    time-weighted averages (the reference's proxy, rlmux/sim.py:69-115):
    a worker's share changes at start / rerate / finish events of
    Training, Reference, PrefillBurst and DecodeLarge nodes; segments shorter than EPS
    are dropped and shares are capped at 1.0 per segment."""
    series = {w: [] for w in workers}
    level = dict.fromkeys(workers, 0.0)
    since = dict.fromkeys(workers, 0.0)
    held = {}

    def cut(w, t):
        if t > since[w] + EPS:
            series[w].append((since[w], t, min(1.0, level[w])))
        since[w] = t

    for ev in events:
        if ev.kind not in ("start", "finish", "rerate"):
            continue
        compute = kind_of(ev.node_id) in COMPUTE_BOUND_KINDS
        share = float(ev.alloc.split("/")[0]) if (compute and ev.alloc != "-") else 0.0
        if ev.kind == "start":
            held[ev.node_id] = share
            if share:
                cut(ev.worker_id, ev.time)
                level[ev.worker_id] += share
        elif ev.kind == "rerate":
            if compute:
                cut(ev.worker_id, ev.time)
                level[ev.worker_id] += share - held.get(ev.node_id, 0.0)
                held[ev.node_id] = share
        else:
            share = held.pop(ev.node_id, 0.0)
            if share:
                cut(ev.worker_id, ev.time)
                level[ev.worker_id] -= share
    avg = {}
    for w in workers:
        cut(w, makespan)
        busy = sum((t1 - t0) * s for t0, t1, s in series[w])
        avg[w] = busy / makespan if makespan > 0 else 0.0
    return avg, series


def simulate(schedule, instance) -> SimulationReport:
    from .state import State

    inst = as_instance(instance)
    st = State(inst, record=True)
    for timed in schedule.actions:
        if timed.start < st.now - 1e-6:
            raise DependencyViolationError(f"action at t={timed.start} recorded after simulated time {st.now}")
        while st.now < timed.start - EPS:
            if not st.has_events():
                st.advance(until=timed.start)
                break
            st.advance(until=timed.start)
        try:
            st.apply(action_from(timed.action))
        except SchedulingError as exc:
            raise DependencyViolationError(str(exc)) from None
    while not st.done():
        if not st.has_events():
            done = st.completion_times()
            pending = sorted(set(st.alive_ids()) - set(done))
            raise DependencyViolationError(f"schedule leaves work unscheduled: {pending[:4]}")
        st.advance()
    pipelines = sorted(g.pipeline_id for g in inst.graphs)
    latency = {p: 0.0 for p in pipelines}
    tokens = {p: 0 for p in pipelines}
    for nid, t in st.completion_times().items():
        node = st.node(nid)
        latency[node.pipeline_id] = max(latency[node.pipeline_id], t)
        tokens[node.pipeline_id] += node.token_total
    total = sum(tokens.values())
    makespan = st.makespan
    events = [TimelineEvent(*e) for e in st.events()]
    alive = {nid: st.node(nid).kind for nid in st.alive_ids()}
    util_avg, util_series = utilization(events, makespan, inst.workers(), alive.get)
    return SimulationReport(makespan=makespan, per_pipeline_latency=latency,
                            per_pipeline_avg_step_latency=dict(latency), per_pipeline_max_step_latency=dict(latency),
                            per_pipeline_tokens=tokens, aggregate_throughput=total / makespan if makespan > 0 else 0.0,
                            utilization_avg=util_avg, utilization_series=util_series, events=events,
                            policy=schedule.policy, metadata=dict(schedule.metadata))
