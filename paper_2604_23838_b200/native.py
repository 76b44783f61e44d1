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
from .encode import InstanceEncoding, StateEncoding
from .model import SchedulingError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RLX_LIB") or os.path.join(HERE, "librlx.so")
_lib = None


class NativeUnavailable(RuntimeError):
    pass


def load_library(path: str = LIB_PATH) -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise NativeUnavailable(f"{path} not built (run `python -m paper_2604_23838_b200.build`)")
        _lib = abi.bind(C.CDLL(path))
        if _lib.rlx_abi_version() != abi.RLX_ABI_VERSION:
            raise NativeUnavailable("librlx.so ABI version mismatch")
    return _lib


def _raise(code: int, msg: str):
    if code == abi.RLX_ERR_SCHEDULING:
        raise SchedulingError(msg)
    if code == abi.RLX_ERR_KEY:
        raise KeyError(msg)
    if code == abi.RLX_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(f"rlx status {code}: {msg}")


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
        self.history = []  # per-decision RlxDecision copies (stats)
        self.record = False
        if instance is not None:
            self.bind(instance)

    def bind(self, instance) -> None:
        self.enc = InstanceEncoding(instance)
        self.senc = StateEncoding(self.enc)
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
        """Score every candidate of `state` on the GPU — or the serial shard
        [b, e) (`shard`), or contiguous block r of w (`part=(r, w)`, sized by
        the library from the candidate count, dist.shard_range)."""
        n_all = self.count(state, window, max_merge) if (want_keys and shard is None) else None
        # encode AFTER count(): every encode() replaces the arrays the previous
        # descriptor points into
        sd = self.senc.encode(state)
        args = abi.RlxDecideArgs()
        args.window = int(window)
        args.max_merge = 0 if max_merge is None else int(max_merge)
        args.serial_begin, args.serial_end = (0, -1) if shard is None else (int(shard[0]), int(shard[1]))
        if part is not None:
            if want_keys:
                raise ValueError("want_keys needs an explicit shard")
            args.serial_begin, args.serial_end = int(part[0]), int(part[1])
            args.flags |= abi.RLX_F_SHARD
        keys = None
        if want_keys:
            n = n_all if shard is None else shard[1] - shard[0]
            keys = np.zeros((max(int(n), 1), 2), dtype=np.float64)
            args.keys_out = keys.ctypes.data_as(C.POINTER(C.c_double))
        args.dev_key_out = dev_key_ptr
        out = abi.RlxDecision()
        rc = self.lib.rlx_decide(self.handle, C.byref(sd), C.byref(args), C.byref(out))
        if rc != 0:
            _raise(rc, self.error())
        self.last = out
        if self.record:
            self.history.append(out)
        if want_keys:
            nk = out.n_candidates if shard is None else min(shard[1], out.n_candidates) - shard[0]
            self.keys = keys[: max(int(nk), 0)]
        return out

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
        """Candidate count of a state (planning only: an empty shard)."""
        sd = self.senc.encode(state)
        args = abi.RlxDecideArgs()
        args.window = int(window)
        args.max_merge = 0 if max_merge is None else int(max_merge)
        args.serial_begin, args.serial_end = 0, 0
        out = abi.RlxDecision()
        rc = self.lib.rlx_decide(self.handle, C.byref(sd), C.byref(args), C.byref(out))
        if rc != 0:
            _raise(rc, self.error())
        return out.n_candidates

    def decode(self, serial: int):
        a = abi.RlxAction()
        rc = self.lib.rlx_decode(self.handle, int(serial), C.byref(a))
        if rc != 0:
            _raise(rc, self.error())
        return self.senc.action_from_raw(a)

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
            action = self.senc.action_from_raw(d.action)
            if log is not None:
                log.append({"now": state.now, "n": d.n_candidates,
                            "key": [d.cost, d.finish, d.priority, d.serial], "action": action})
            return action

        return choose
