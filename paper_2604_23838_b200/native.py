"""Python side of the C-ABI: loads the in-tree `librlx.so` and exposes the
device chooser.

There is deliberately no fallback: if the library or a CUDA device is
missing, `Evaluator` raises `NativeUnavailable` instead of scoring on the
CPU.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi
from .encode import instance_encoding
from .model import SchedulingError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RLX_LIB") or os.path.join(HERE, "librlx.so")
_lib = None


class NativeUnavailable(RuntimeError):
    pass


def load_library(path: str = LIB_PATH, require_device: bool = True) -> C.CDLL:
    """The in-tree CUDA library. Loading needs no device (the native
    execution state and the host planner run without one); scoring does
    (`Evaluator` raises NativeUnavailable when rlx_open finds no GPU)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise NativeUnavailable(f"{path} not built (run `python -m paper_2604_23838_b200.build`)")
        _lib = abi.bind(C.CDLL(path))
        if _lib.rlx_abi_version() != abi.RLX_ABI_VERSION:
            raise NativeUnavailable("librlx.so ABI version mismatch")
    return _lib


class CapacityError(RuntimeError):
    """The input exceeds a compiled limit of this build (RLX_ERR_LIMIT,
    include/rlx.h); the reference itself has no such limit. INTEGRATION.md §4
    lists them."""


def _raise(code: int, msg: str, serial: int | None = None):
    """Status code -> the reference's exception class. A failing candidate's
    serial rides on the exception (`.serial`), the message is the
    reference's text."""
    if code == abi.RLX_ERR_SCHEDULING:
        exc = SchedulingError(msg)
    elif code == abi.RLX_ERR_KEY:
        exc = KeyError(msg)
    elif code == abi.RLX_ERR_VALUE:
        exc = ValueError(msg)
    elif code == abi.RLX_ERR_LIMIT:
        exc = CapacityError(msg)
    else:
        exc = RuntimeError(f"rlx status {code}: {msg}")
    exc.serial = serial
    exc.code = code
    raise exc


def raise_device_error(code: int, serial: int | None = None):
    """Raise the reference's exception for a device error code (the low byte
    of RlxDecision.err_key): the same class and text on every rank."""
    lib = load_library(require_device=False)
    buf = C.create_string_buffer(512)
    st = lib.rlx_error_text(int(code), buf, 512)
    _raise(st, buf.value.decode(), serial)


def plan_info(state, window: int, max_merge: int | None = None) -> abi.RlxPlanInfo:
    """Host-only planning of `state`'s decision (rlx_plan_info): candidate
    counts and plan sizes, or the CapacityError the device path would
    raise. Needs no GPU."""
    lib = load_library(require_device=False)
    out = abi.RlxPlanInfo()
    err = C.create_string_buffer(512)
    sd = state.snapshot()
    rc = lib.rlx_plan_info(C.byref(state.enc.desc), C.byref(sd), int(window),
                           0 if max_merge is None else int(max_merge), C.byref(out), err, 512)
    if rc != 0:
        _raise(rc, err.value.decode())
    return out


class Evaluator:
    """One GPU handle bound to one instance (rlx_open + rlx_load_instance)."""

    def __init__(self, instance=None, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.rlx_open(int(device), C.byref(h))
        if rc != 0:
            raise NativeUnavailable(f"rlx_open(device={device}) failed with status {rc} (no CUDA device?)")
        self.handle = h
        self.device = device
        self.instance = None
        self.last = None
        self.last_state = None
        self.n_decisions = 0
        self.history = []  # per-decision RlxDecision copies (stats)
        self.record = False
        if instance is not None:
            self.bind(instance)

    def bind(self, instance) -> None:
        self.enc = instance_encoding(instance)
        rc = self.lib.rlx_load_instance(self.handle, C.byref(self.enc.desc))
        if rc != 0:
            _raise(rc, self.error())
        self.instance = instance

    def error(self) -> str:
        return (self.lib.rlx_last_error(self.handle) or b"").decode()

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.rlx_close(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def decide(self, state, window: int, max_merge: int | None = None, shard=None, want_keys=False,
               dev_key_ptr: int | None = None, part=None) -> abi.RlxDecision:
        """Score every candidate of `state` (a `state.State`) on the GPU —
        or the serial shard [b, e) (`shard`, e < 0: to the last candidate),
        or cost-balanced part r of w (`part=(r, w)`, dist.py)."""
        self._check_state(state)
        args = abi.RlxDecideArgs()
        args.window = int(window)
        args.max_merge = 0 if max_merge is None else int(max_merge)
        b, e = (0, -1) if shard is None else (int(shard[0]), int(shard[1]))
        if part is not None:
            if want_keys:
                raise ValueError("want_keys needs an explicit shard")
            args.serial_begin, args.serial_end = int(part[0]), int(part[1])
            args.flags |= abi.RLX_F_SHARD
        keys = None
        if want_keys:
            if e < 0 or b < 0:  # resolve "to the last candidate" before sizing the buffer
                n = plan_info(state, window, max_merge).n_candidates
                b = max(b, 0)
                e = n if e < 0 else e
            keys = np.zeros((max(e - b, 1), 2), dtype=np.float64)
            args.keys_out = keys.ctypes.data_as(C.POINTER(C.c_double))
        if part is None:
            args.serial_begin, args.serial_end = b, e
        args.dev_key_out = dev_key_ptr
        sd = state.snapshot()
        out = abi.RlxDecision()
        rc = self.lib.rlx_decide(self.handle, C.byref(sd), C.byref(args), C.byref(out))
        self.last_n_candidates = out.n_candidates
        if rc != 0:
            _raise(rc, self.error(), out.serial if out.serial >= 0 else None)
        self.last = out
        self.last_state = state
        if self.record:
            self.history.append(out)
        if want_keys:
            nk = min(e, out.n_candidates) - b
            self.keys = keys[: max(int(nk), 0)]
        return out

    def _check_state(self, state) -> None:
        if state.instance is not self.instance and state.enc is not self.enc:
            raise ValueError("the state belongs to a different instance than this Evaluator is bound to")

    def schedule(self, state, window: int, max_merge: int | None = None, max_decisions: int | None = None):
        """The whole decision loop (`_drive`, scheduler.py:925-950) behind
        one C call (rlx_drive): plan -> score -> argmin -> apply the winner to
        the native `state` -> advance, until done. Returns the RlxStep
        records (applied actions, their keys and decision latencies);
        `state.replay_steps` turns them into actions."""
        self._check_state(state)
        info = state.info()
        cap = 2 * info.n_total + 8
        steps = (abi.RlxStep * cap)()
        args = abi.RlxDriveArgs()
        args.window = int(window)
        args.max_merge = 0 if max_merge is None else int(max_merge)
        args.max_decisions = 0 if max_decisions is None else int(max_decisions)
        args.max_steps = cap
        n_steps = C.c_int64()
        n_dec = C.c_int64()
        rc = self.lib.rlx_drive(self.handle, state.handle, C.byref(args), steps, C.byref(n_steps), C.byref(n_dec))
        done = list(steps[: n_steps.value])
        self.n_decisions = n_dec.value
        if rc != 0:
            state.replay_steps(done)  # keep the id mirror in step with the native state
            _raise(rc, self.error())
        return done

    def rescore(self, window: int, shard=None, dev_key_ptr: int | None = None, part=None) -> abi.RlxDecision:
        """Re-run scoring + argmin on the plan already resident on the device
        (RLX_F_REUSE_PLAN): the device-only part of the last `decide`."""
        args = abi.RlxDecideArgs()
        args.window = int(window)
        args.serial_begin, args.serial_end = (0, -1) if shard is None else (int(shard[0]), int(shard[1]))
        args.dev_key_out = dev_key_ptr
        args.flags = abi.RLX_F_REUSE_PLAN
        if part is not None:
            args.serial_begin, args.serial_end = int(part[0]), int(part[1])
            args.flags |= abi.RLX_F_SHARD
        out = abi.RlxDecision()
        rc = self.lib.rlx_decide(self.handle, None, C.byref(args), C.byref(out))
        if rc != 0:
            _raise(rc, self.error())
        self.last = out
        return out

    def set_stream(self, stream_ptr: int | None) -> None:
        """Issue the handle's work on a caller CUDA stream (e.g. torch's
        current stream, so torch CUDA events and NCCL order with it)."""
        rc = self.lib.rlx_set_stream(self.handle, stream_ptr or None)
        if rc != 0:
            _raise(rc, self.error())

    def count(self, state, window: int, max_merge: int | None = None) -> int:
        """Candidate count of a state (host planning only)."""
        return plan_info(state, window, max_merge).n_candidates

    def decode(self, serial: int):
        """Serial of the last decided state -> its action."""
        a = abi.RlxAction()
        rc = self.lib.rlx_decode(self.handle, int(serial), C.byref(a))
        if rc != 0:
            _raise(rc, self.error())
        return self.last_state.action_from_raw(a)

    def chooser(self, window: int, max_merge: int | None = None, log=None, group=None):
        """A `drive` chooser deciding on this GPU (or, with a process group,
        on this rank's shard followed by the cross-GPU min-loc)."""
        if group is not None:
            from .dist import ShardedChooser

            return ShardedChooser(self, window, max_merge, group, log)

        def choose(state):
            d = self.decide(state, window, max_merge)
            if d.n_candidates == 0:
                return None
            action = state.action_from_raw(d.action)
            if log is not None:
                log.append({"now": state.now, "n": d.n_candidates,
                            "key": [d.cost, d.finish, d.priority, d.serial], "action": action})
            return action

        return choose
