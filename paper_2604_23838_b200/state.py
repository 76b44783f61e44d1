"""The decision loop's execution state, held natively in librlx.so.

`State(instance, record=False)` is the reference's `ExecState`
(rlmux/scheduler.py:339-634) behind the C-ABI (include/rlx.h
rlx_state_*): readiness, apply with its validation errors, merge surgery,
advance with survivor re-rating, tool-wait auto-start. It lives on the
library's structure-of-arrays (csrc/rlx_state.cpp), so the per-decision
input of the device chooser is a view of those arrays (`snapshot`) rather
than a Python re-encode, and the whole `_drive` loop can run behind one
C call (`Evaluator.schedule`).

This module only translates between node ids and the native node indices
and computes the slowdown factors of user-supplied allocations (prelude
actions) with the instance's model; the state itself never lives here.
"""

from __future__ import annotations

import ctypes as C

from . import abi
from .encode import instance_encoding
from .model import (
    KIND_ORDER,
    Exclusive,
    Merge,
    Multiplex,
    SchedulingError,
    SubStage,
    complement_allocation,
)


def _lib():
    from .native import load_library

    return load_library(require_device=False)


def _raise(code: int, msg: str, exc: BaseException | None = None):
    if code == abi.RLX_ERR_SCHEDULING:
        raise SchedulingError(msg)
    if code == abi.RLX_ERR_KEY:
        if exc is not None:
            raise exc
        raise KeyError(msg)
    if code == abi.RLX_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(f"rlx status {code}: {msg}")


class State:
    """ExecState over an instance's combined sub-stage graphs (native)."""

    def __init__(self, instance, record: bool = False, _clone_of: "State | None" = None):
        self.lib = _lib()
        self.instance = instance
        self.enc = instance_encoding(instance)
        self.record = record
        h = C.c_void_p()
        if _clone_of is None:
            rc = self.lib.rlx_state_create(C.byref(self.enc.desc), C.byref(self.enc.graph.desc), 1 if record else 0,
                                           C.byref(h))
            self.handle = h
            if rc != 0:
                _raise(rc, self.lib.rlx_state_error(h).decode())
            self._ids = list(self.enc.graph.ids)  # state index -> id
            self._index = dict(self.enc.graph.index)  # id -> state index (alive and dead)
            self._order = list(range(len(self._ids)))  # alive nodes, dict order (= snapshot order)
        else:
            rc = self.lib.rlx_state_clone(_clone_of.handle, C.byref(h))
            self.handle = h
            if rc != 0:
                raise RuntimeError("rlx_state_clone failed")
            self._ids = list(_clone_of._ids)
            self._index = dict(_clone_of._index)
            self._order = list(_clone_of._order)
        self._snap = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.rlx_state_destroy(h)
            self.handle = None

    def clone(self) -> "State":
        return State(self.instance, record=False, _clone_of=self)

    # -- queries ----------------------------------------------------------

    def info(self) -> abi.RlxStateInfo:
        out = abi.RlxStateInfo()
        self.lib.rlx_state_info(self.handle, C.byref(out))
        return out

    @property
    def now(self) -> float:
        return self.info().now

    @property
    def makespan(self) -> float:
        return self.info().makespan

    def done(self) -> bool:
        return bool(self.info().done)

    def has_events(self) -> bool:
        return bool(self.info().has_events)

    def node_info(self, idx: int) -> abi.RlxNodeInfo:
        out = abi.RlxNodeInfo()
        if self.lib.rlx_state_node(self.handle, int(idx), C.byref(out)) != 0:
            raise IndexError(idx)
        return out

    def alive_ids(self) -> list:
        """Alive node ids in the reference's dict order."""
        return [self._ids[i] for i in self._order]

    def completion_times(self) -> dict:
        """completion_time of every completed alive node (scheduler.py:438)."""
        n = len(self._ids)
        done = (C.c_uint8 * n)()
        times = (C.c_double * n)()
        self.lib.rlx_state_completion(self.handle, done, times)
        return {self._ids[i]: times[i] for i in self._order if done[i]}

    def node(self, nid: str) -> SubStage:
        """The SubStage of an alive node (merged nodes are rebuilt from the
        native record; their sample_ids are the union of the members')."""
        i = self._index[nid]
        for g in self.instance.graphs:
            if nid in g.nodes:
                return g.nodes[nid]
        x = self.node_info(i)
        return SubStage(id=nid, pipeline_id=self.enc.pipe_ids[x.pipe], worker_id=self.enc.workers[x.worker],
                        kind=KIND_ORDER[x.kind], duration=x.duration, mem_fraction=x.mem,
                        step_span=(x.span_lo, x.span_hi), remaining_decode_tokens=x.remaining,
                        active_requests=x.active, context_tokens=x.context, token_total=x.token_total)

    def events(self) -> list:
        """Recorded events as (time, worker_id, kind, node_id, alloc) tuples,
        the reference's format (scheduler.py:389-391)."""
        n = self.info().n_events
        buf = (abi.RlxEvent * max(n, 1))()
        self.lib.rlx_state_events(self.handle, 0, n, buf)
        out = []
        for e in buf[:n]:
            alloc = "-" if e.sm != e.sm else f"{e.sm:.4f}/{e.mem:.4f}"
            out.append((e.time, self.enc.workers[e.worker], abi.EVENT_NAMES[e.kind], self._ids[e.node], alloc))
        return out

    # -- the device chooser's input ----------------------------------------

    def snapshot(self) -> abi.RlxStateDesc:
        """RlxStateDesc view of the native arrays (valid until the next mutation)."""
        d = abi.RlxStateDesc()
        self.lib.rlx_state_snapshot(self.handle, C.byref(d))
        d._owner = self
        return d

    def action_from_raw(self, a: abi.RlxAction, space: str = "snapshot"):
        """RlxAction -> Exclusive / Multiplex / Merge; node indices are
        snapshot indices (rlx_decide) or state indices (rlx_drive)."""
        ids = (lambda i: self._ids[self._order[i]]) if space == "snapshot" else (lambda i: self._ids[i])
        if a.cls == abi.CLASS_EXCLUSIVE:
            return Exclusive(ids(a.node_a))
        if a.cls == abi.CLASS_MULTIPLEX:
            return Multiplex(ids(a.node_a), ids(a.node_b), self.enc.allocs[a.alloc])
        return Merge(tuple(ids(a.members[i]) for i in range(a.n_members)), self.enc.workers[a.target_worker])

    # -- mutation -----------------------------------------------------------

    def _idx(self, nid: str) -> int:
        i = self._index.get(nid)
        if i is None or i not in self._alive_set():
            raise SchedulingError(f"unknown sub-stage {nid!r}")
        return i

    def _alive_set(self):
        if self._snap is None or self._snap[0] is not self._order:
            self._snap = (self._order, set(self._order))
        return self._snap[1]

    def _rate(self, kind, partner, alloc):
        try:
            return self.instance.model.slowdown(kind, partner, alloc), None
        except KeyError as exc:
            return float("nan"), exc

    def apply(self, action) -> None:
        a = abi.RlxApply()
        exc = None
        name = type(action).__name__
        if name == "Exclusive":
            i = self._idx(action.node_id)
            a.cls = abi.CLASS_EXCLUSIVE
            a.node_a = i
            kind = KIND_ORDER[self.node_info(i).kind]
            a.rate_a, exc = self._rate(kind, None, action.alloc)
            a.sm_a, a.mem_a = action.alloc.sm_share, action.alloc.mem_share
        elif name == "Multiplex":
            i, j = self._idx(action.node_a), self._idx(action.node_b)
            a.cls = abi.CLASS_MULTIPLEX
            a.node_a, a.node_b = i, j
            ka, kb = KIND_ORDER[self.node_info(i).kind], KIND_ORDER[self.node_info(j).kind]
            alloc_b = complement_allocation(action.alloc_a, self.instance.headroom)
            a.rate_a, exc = self._rate(ka, kb, action.alloc_a)
            if exc is None:
                a.rate_b, exc = self._rate(kb, ka, alloc_b)
            else:
                a.rate_b = float("nan")
            a.sm_a, a.mem_a = action.alloc_a.sm_share, action.alloc_a.mem_share
            a.sm_b, a.mem_b = alloc_b.sm_share, alloc_b.mem_share
        elif name == "Merge":
            ids = tuple(action.member_ids)
            if len(ids) > abi.RLX_MAX_MEMBERS:
                raise RuntimeError(f"rlx status {abi.RLX_ERR_LIMIT}: merge sets above 64 members")
            if len(ids) < 2:
                raise SchedulingError("merge needs at least two fragments")
            a.cls = abi.CLASS_MERGE
            a.n_members = len(ids)
            for k, nid in enumerate(ids):
                a.members[k] = self._idx(nid)
            w = self.enc.worker_index.get(action.target_worker)
            a.target_worker = -1 if w is None else w
        else:
            raise SchedulingError(f"unknown action {action!r}")
        rc = self.lib.rlx_state_apply(self.handle, C.byref(a))
        if rc != 0:
            _raise(rc, self.lib.rlx_state_error(self.handle).decode(), exc)
        if name == "Merge":
            self._note_merge(ids, action.target_worker)

    def _note_merge(self, ids, target_worker) -> None:
        mid = "merge[" + "+".join(ids) + f"]@w{target_worker}"
        gone = {self._index[x] for x in ids}
        self._order = [i for i in self._order if i not in gone]
        self._index[mid] = len(self._ids)
        self._order.append(len(self._ids))
        self._ids.append(mid)

    def replay_steps(self, steps) -> list:
        """Mirror the id bookkeeping of actions the library applied
        (rlx_drive) and return them as actions."""
        out = []
        for st in steps:
            act = self.action_from_raw(st.action, space="state")
            if isinstance(act, Merge):
                self._note_merge(act.member_ids, act.target_worker)
            out.append((st.start, act))
        return out

    def enumerate_raw(self) -> list:
        """enumerate_actions (scheduler.py:648-703) of this state, natively:
        RlxAction records in serial order (node indices = state indices)."""
        n = C.c_int64()
        self.lib.rlx_enumerate(C.byref(self.enc.desc), self.handle, None, 0, C.byref(n))
        buf = (abi.RlxAction * max(n.value, 1))()
        self.lib.rlx_enumerate(C.byref(self.enc.desc), self.handle, buf, n.value, C.byref(n))
        return list(buf[: n.value])

    def run_to_completion(self) -> None:
        """ExecState.run_to_completion (scheduler.py:629-634)."""
        while not self.done():
            if not self.has_events():
                done = self.completion_times()
                stuck = sorted(set(self.alive_ids()) - set(done))
                raise SchedulingError(f"stuck with nothing running; pending: {stuck[:4]}")
            self.advance()

    def advance(self, until: float | None = None) -> None:
        rc = self.lib.rlx_state_advance(self.handle, 0 if until is None else 1, 0.0 if until is None else float(until))
        if rc != 0:
            _raise(rc, self.lib.rlx_state_error(self.handle).decode())
