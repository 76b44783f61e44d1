"""Replay of a Schedule into the headline metrics (rlmux/sim.py:118-173).

Used to check the north-star parity clause "fp64 makespan and throughput
estimates agree within 1e-9 relative": the schedule produced by the GPU
chooser is re-executed on the host engine and reduced to makespan,
per-pipeline latency, tokens and aggregate throughput exactly as the
reference's `simulate` does.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .engine import HostState
from .instance_io import action_from, as_instance
from .model import EPS, SchedulingError


class DependencyViolationError(ValueError):
    """rlmux/sim.py:37"""


@dataclass
class SimulationReport:
    makespan: float
    per_pipeline_latency: dict
    per_pipeline_tokens: dict
    aggregate_throughput: float
    events: list = field(default_factory=list)
    policy: str = ""
    metadata: dict = field(default_factory=dict)

    @property
    def total_tokens(self) -> int:
        return sum(self.per_pipeline_tokens.values())


def simulate(schedule, instance) -> SimulationReport:
    inst = as_instance(instance)
    st = HostState(inst, record=True)
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
            pending = sorted(set(st.nodes) - st.completed)
            raise DependencyViolationError(f"schedule leaves work unscheduled: {pending[:4]}")
        st.advance()
    pipelines = sorted(g.pipeline_id for g in inst.graphs)
    latency = {p: 0.0 for p in pipelines}
    tokens = {p: 0 for p in pipelines}
    for nid, t in st.completion_time.items():
        node = st.nodes[nid]
        latency[node.pipeline_id] = max(latency[node.pipeline_id], t)
        tokens[node.pipeline_id] += node.token_total
    total = sum(tokens.values())
    makespan = st.makespan
    return SimulationReport(makespan=makespan, per_pipeline_latency=latency, per_pipeline_tokens=tokens,
                            aggregate_throughput=total / makespan if makespan > 0 else 0.0,
                            events=list(st.events), policy=schedule.policy, metadata=dict(schedule.metadata))
