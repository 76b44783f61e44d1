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
