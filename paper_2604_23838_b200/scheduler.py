"""Reference-compatible scheduling entry points on the B200 evaluator.

`lookahead_schedule(instance, window=3, prelude=(), *, max_merge=None)` and
`greedy_schedule(instance, prelude=())` keep the signatures, return types
and error behaviour of rlmux/scheduler.py:953-980. The decision loop is
the reference's `_drive` (:925-950): enumerate -> choose -> apply until no
candidate is left, then advance simulated time. The chooser is the hot
path and runs entirely on the GPU through the C-ABI (`native.Evaluator`):
candidate generation, the W-round look-ahead list-scheduling passes,
merge follow-ups, finish estimates and the (cost, finish, priority,
serial) argmin. There is no CPU scoring path: if the CUDA library cannot
be loaded the call raises.

Passing an `rlmux.Instance` works too: it is converted on the way in and
the returned Schedule is re-expressed with rlmux's action classes, so it
can be handed straight back to `rlmux.sim.simulate`.
"""

from __future__ import annotations

import importlib

from .instance_io import action_as, action_from, as_instance, is_reference_instance
from .model import Schedule, SchedulingError, TimedAction
from .state import State


def drive(instance, chooser, policy: str, metadata: dict, prelude=()) -> Schedule:
    """The reference decision loop (rlmux/scheduler.py:925-950) with a
    Python chooser over the native state (used by the multi-GPU chooser,
    dist.ShardedChooser, and by tests with the CPU oracle's chooser). The
    single-GPU path runs this loop inside the library (`lookahead_schedule`
    -> Evaluator.schedule -> rlx_drive).

    `chooser(state)` returns the action to apply now, or None when there is
    no candidate (the reference's `chooser(state, cands) if cands else None`).
    """
    state = State(instance)
    actions = []
    for action in prelude:
        actions.append(TimedAction(state.now, action))
        state.apply(action)
    while not state.done():
        while True:
            action = chooser(state)
            if action is None:
                break
            actions.append(TimedAction(state.now, action))
            state.apply(action)
        if state.done():
            break
        if not state.has_events():
            raise SchedulingError(f"{policy}: stalled with no running work")
        state.advance()
    return Schedule(actions=actions, policy=policy, metadata=metadata)


def _ref_schedule_module(x):
    return importlib.import_module(type(x).__module__.rsplit(".", 1)[0] + ".scheduler")


def lookahead_schedule(instance, window: int = 3, prelude=(), *, max_merge: int | None = None,
                       evaluator=None) -> Schedule:
    """Pick, at each decision point, the candidate minimising
    (window cost, own finish, priority, serial) — scored on the GPU."""
    if window < 1:
        raise ValueError("window must be >= 1")
    ref = is_reference_instance(instance)
    inst = as_instance(instance)
    pre = tuple(action_from(a) for a in prelude)
    from .native import Evaluator

    ev = evaluator if evaluator is not None else Evaluator(inst)
    if ev.instance is not inst:
        ev.bind(inst)
    state = State(inst)
    actions = []
    for action in pre:
        actions.append(TimedAction(state.now, action))
        state.apply(action)
    steps = ev.schedule(state, window, max_merge)  # the _drive loop, natively
    actions += [TimedAction(t, a) for t, a in state.replay_steps(steps)]
    sched = Schedule(actions=actions, policy="lookahead", metadata={"window": str(window)})
    if ref:
        mod = _ref_schedule_module(instance)
        sched = mod.Schedule(actions=[mod.TimedAction(t.start, action_as(t.action, mod)) for t in sched.actions],
                             policy=sched.policy, metadata=sched.metadata)
    return sched


def greedy_schedule(instance, prelude=(), *, max_merge: int | None = None, evaluator=None) -> Schedule:
    """Window-1 look-ahead (rlmux/scheduler.py:977-980)."""
    sched = lookahead_schedule(instance, window=1, prelude=prelude, max_merge=max_merge, evaluator=evaluator)
    return type(sched)(actions=sched.actions, policy="greedy", metadata={})


def serial_schedule(instance) -> Schedule:
    """Temporal multiplexing, pipelines back to back (rlmux/scheduler.py:983-1006):
    at each decision the first Exclusive candidate (enumerate_actions order)
    of the first pipeline, by id, with work left. A brute-force seed."""
    inst = as_instance(instance)
    order = sorted(g.pipeline_id for g in inst.graphs)
    own = {g.pipeline_id: set(g.nodes) for g in inst.graphs}
    pipe_of = {nid: g.pipeline_id for g in inst.graphs for nid in g.nodes}

    def chooser(state):
        alive = set(state.alive_ids())
        done = state.completion_times()
        active = next((pid for pid in order if any(n not in done for n in own[pid] & alive)), None)
        if active is None:
            return None
        for a in state.enumerate_raw():
            if a.cls == 2:  # Exclusive
                act = state.action_from_raw(a, space="state")
                if pipe_of.get(act.node_id) == active:
                    return act
        return None

    sched = drive(inst, chooser, "serial", {})
    return _as_caller(instance, sched)


def brute_force_schedule(instance, node_limit: int = 10, *, _seeds=None) -> Schedule:
    """Exhaustive search over action sequences (including idling) for the
    minimal makespan under the engine semantics (rlmux/scheduler.py:1148-1218).
    Seeds: the look-ahead (device), greedy (device) and serial schedules'
    best makespan; the depth-first branch-and-bound runs natively
    (rlx_branch_and_bound) in the reference's visiting order, so the
    returned schedule is the reference's. `_seeds` (tests) replaces the
    seed schedules."""
    import ctypes as C

    from . import abi
    from .encode import instance_encoding
    from .model import EPS, OracleLimitError
    from .native import _raise, load_library

    inst = as_instance(instance)
    total = sum(len(g.nodes) for g in inst.graphs)
    if total > node_limit:
        raise OracleLimitError(f"instance has {total} sub-stages, above the limit of {node_limit}; "
                               "use the look-ahead scheduler for larger instances")
    best_make, best_actions = float("inf"), []
    seeds = _seeds if _seeds is not None else (lambda i: lookahead_schedule(i), greedy_schedule, serial_schedule)
    for seed in seeds:
        try:
            sched = seed(inst) if callable(seed) else seed
        except SchedulingError:
            continue
        state = State(inst)
        for timed in sched.actions:
            a = action_from(timed.action)
            state.advance(until=timed.start)
            while state.now < timed.start - EPS:
                state.advance(until=timed.start)
            state.apply(a)
        state.run_to_completion()
        if state.makespan < best_make:
            best_make = state.makespan
            best_actions = [TimedAction(t.start, action_from(t.action)) for t in sched.actions]
    enc = instance_encoding(inst)
    lib = load_library(require_device=False)
    cap = 4 * total + 16
    steps = (abi.RlxStep * cap)()
    n = C.c_int32()
    best = C.c_double()
    visited = C.c_int64()
    rc = lib.rlx_branch_and_bound(C.byref(enc.desc), C.byref(enc.graph.desc), float(best_make), cap, steps,
                                  C.byref(n), C.byref(best), C.byref(visited))
    if rc != 0:
        _raise(rc, "branch-and-bound failed")
    if n.value >= 0:
        replay = State(inst)
        best_actions = [TimedAction(t, a) for t, a in replay.replay_steps(steps[: n.value])]
    sched = Schedule(actions=best_actions, policy="oracle", metadata={"limit": str(node_limit)})
    return _as_caller(instance, sched)


def _as_caller(instance, sched: Schedule):
    """Re-express a Schedule with the caller's classes (rlmux objects in, rlmux out)."""
    if not is_reference_instance(instance):
        return sched
    mod = _ref_schedule_module(instance)
    return mod.Schedule(actions=[mod.TimedAction(t.start, action_as(t.action, mod)) for t in sched.actions],
                        policy=sched.policy, metadata=sched.metadata)
