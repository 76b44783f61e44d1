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


def simulate_batch(schedules, instance, threads: int | None = None) -> list:
    """`simulate` for many schedules of one instance:
    every schedule is replayed on its own copy of the native ExecState in
    librlx.so (csrc/rlx_sim.cpp), over `threads` host threads (default: all),
    with the metrics folded natively in the reference's operation order.
    The reports equal `simulate`'s field for field except `events` and
    `utilization_series`, which stay empty (the batch keeps only the
    averages). A schedule whose allocations fall outside the instance's
    slowdown LUT is replayed by `simulate` instead. The first failing
    schedule raises the exception `simulate` would raise for it."""
    import ctypes as C

    from . import abi
    from .encode import instance_encoding
    from .model import Exclusive, Multiplex
    from .native import load_library

    inst = as_instance(instance)
    enc = instance_encoding(inst)
    lib = load_library(require_device=False)
    scheds = list(schedules)
    acts, blob, off = [], bytearray(), [0]
    for sched in scheds:
        for timed in sched.actions:
            a = action_from(timed.action)
            x = abi.RlxSimAction()
            x.start = float(timed.start)
            if isinstance(a, Exclusive):
                ids = [a.node_id]
                x.cls, x.sm, x.mem = abi.CLASS_EXCLUSIVE, a.alloc.sm_share, a.alloc.mem_share
            elif isinstance(a, Multiplex):
                ids = [a.node_a, a.node_b]
                x.cls, x.sm, x.mem = abi.CLASS_MULTIPLEX, a.alloc_a.sm_share, a.alloc_a.mem_share
            else:
                ids = list(a.member_ids)
                x.cls, x.target_worker = abi.CLASS_MERGE, int(a.target_worker)
            x.n_ids, x.id_off = len(ids), len(blob)
            for nid in ids:
                blob += nid.encode() + b"\0"
            acts.append(x)
        off.append(len(acts))
    n = len(scheds)
    P, W = len(inst.graphs), len(enc.workers)
    res = (abi.RlxSimResult * max(n, 1))()
    lat = (C.c_double * max(n * P, 1))()
    tok = (C.c_int64 * max(n * P, 1))()
    util = (C.c_double * max(n * W, 1))()
    arr = (abi.RlxSimAction * max(len(acts), 1))(*acts)
    offs = (C.c_int64 * (n + 1))(*off)
    rc = lib.rlx_simulate_batch(C.byref(enc.desc), C.byref(enc.graph.desc), n, offs, arr, bytes(blob) + b"\0",
                                0 if threads is None else int(threads), res, lat, tok, util)
    if rc != 0 and n:
        raise RuntimeError(f"rlx status {rc}: {res[0].error.decode()}")
    pipes = [g.pipeline_id for g in inst.graphs]
    order = sorted(range(P), key=lambda q: pipes[q])
    out = []
    for s, sched in enumerate(scheds):
        r = res[s]
        if r.status == abi.RLX_ERR_LIMIT:
            out.append(simulate(sched, inst))
            continue
        if r.status != 0:
            msg = r.error.decode()
            if r.status == abi.RLX_ERR_SCHEDULING:
                raise DependencyViolationError(msg)
            if r.status == abi.RLX_ERR_KEY:
                raise KeyError(msg)
            raise RuntimeError(f"rlx status {r.status}: {msg}")
        latency = {pipes[q]: lat[s * P + q] for q in order}
        tokens = {pipes[q]: tok[s * P + q] for q in order}
        util_avg = {enc.workers[w]: util[s * W + w] for w in range(W)}
        out.append(SimulationReport(makespan=r.makespan, per_pipeline_latency=latency,
                                    per_pipeline_avg_step_latency=dict(latency),
                                    per_pipeline_max_step_latency=dict(latency), per_pipeline_tokens=tokens,
                                    aggregate_throughput=r.throughput, utilization_avg=util_avg,
                                    utilization_series={}, events=[], policy=sched.policy,
                                    metadata=dict(sched.metadata)))
    return out
