"""ctypes front-end of the CPU oracle (oracle/rlx_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs — never by the product.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2604_23838_b200 import abi
from paper_2604_23838_b200.encode import instance_encoding

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "librlx_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.oracle_decide.restype = C.c_int
        L.oracle_decide.argtypes = [
            C.POINTER(abi.RlxInstanceDesc), C.POINTER(abi.RlxStateDesc), C.c_int, C.c_int,
            C.POINTER(C.c_int64), C.c_int64, C.c_int, C.POINTER(C.c_double),
            C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double),
            C.POINTER(C.c_int), C.c_char_p, C.c_int,
        ]
        L.oracle_candidate.restype = C.c_int
        L.oracle_candidate.argtypes = [C.POINTER(abi.RlxInstanceDesc), C.POINTER(abi.RlxStateDesc), C.c_int,
                                       C.c_int64, C.POINTER(C.c_int32), C.c_char_p, C.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class Oracle:
    """Scores decision states exactly like the reference chooser."""

    def __init__(self, instance, nthreads: int | None = None):
        self.enc = instance_encoding(instance)
        self.nthreads = nthreads or os.cpu_count() or 1

    def score(self, state, window: int, max_merge: int | None = None, serials=None, want_keys=False):
        """Returns dict(n, best=(cost, finish, prio, serial) or None, keys=ndarray[k,2] or None)."""
        n_all = None
        if want_keys and serials is None:
            # the count first: every encode() replaces the arrays an earlier descriptor points into
            n_all = self.score(state, window, max_merge, serials=[], want_keys=False)["n"]
        sd = state.snapshot()
        mm = 0 if max_merge is None else int(max_merge)
        ser = None
        nser = 0
        if serials is not None:
            ser_arr = np.ascontiguousarray(np.asarray(serials, dtype=np.int64))
            ser = ser_arr.ctypes.data_as(C.POINTER(C.c_int64))
            nser = len(ser_arr)
        keys = None
        kp = None
        if want_keys:
            n_hint = nser if serials is not None else None
            if n_hint is None:
                n_hint = n_all
            keys = np.zeros((max(n_hint, 1), 2), dtype=np.float64)
            kp = keys.ctypes.data_as(C.POINTER(C.c_double))
        if serials is not None and nser == 0:
            ser_arr = np.zeros(1, dtype=np.int64)
            ser = ser_arr.ctypes.data_as(C.POINTER(C.c_int64))
        n = C.c_int64()
        bs = C.c_int64()
        bc = C.c_double()
        bf = C.c_double()
        bp = C.c_int()
        err = C.create_string_buffer(256)
        rc = lib().oracle_decide(C.byref(self.enc.desc), C.byref(sd), int(window), mm, ser, nser, self.nthreads,
                                 kp, C.byref(n), C.byref(bs), C.byref(bc), C.byref(bf), C.byref(bp), err, 256)
        if rc != 0:
            raise OracleError(rc, err.value.decode())
        best = None if bs.value < 0 else (bc.value, bf.value, bp.value, bs.value)
        out = {"n": n.value, "best": best}
        if want_keys:
            out["keys"] = keys[: (nser if serials is not None else n.value)]
        return out

    def candidate(self, state, serial: int, max_merge: int | None = None):
        sd = state.snapshot()
        buf = (C.c_int32 * (6 + abi.RLX_MAX_MEMBERS))()
        err = C.create_string_buffer(256)
        rc = lib().oracle_candidate(C.byref(self.enc.desc), C.byref(sd), 0 if max_merge is None else int(max_merge),
                                    int(serial), buf, err, 256)
        if rc != 0:
            raise OracleError(rc, err.value.decode())
        a = abi.RlxAction()
        a.cls, a.node_a, a.node_b, a.alloc, a.target_worker, a.n_members = buf[:6]
        for i in range(a.n_members):
            a.members[i] = buf[6 + i]
        return state.action_from_raw(a)

    def counts(self, state, window: int, max_merge: int | None = None):
        """(n_multiplex, n_merge, n_exclusive) of a decision: the serial
        space is laid out in that class order (scheduler.py:648-703), so the
        class boundaries are found by binary search on decoded serials."""
        n = self.score(state, window, max_merge, serials=[])["n"]

        def cls(s):
            a = self.candidate(state, s, max_merge)
            name = type(a).__name__
            return 0 if name == "Multiplex" else (1 if name == "Merge" else 2)

        def first(at_least):
            lo, hi = 0, n
            while lo < hi:
                mid = (lo + hi) // 2
                if cls(mid) >= at_least:
                    hi = mid
                else:
                    lo = mid + 1
            return lo

        a, b = first(1), first(2)
        return a, b - a, n - b

    def chooser(self, window: int, max_merge: int | None = None, log=None):
        """A `drive` chooser that decides with the oracle."""

        def choose(state):
            r = self.score(state, window, max_merge)
            if r["n"] == 0:
                return None
            action = self.candidate(state, r["best"][3], max_merge)
            if log is not None:
                log.append({"now": state.now, "n": r["n"], "key": list(r["best"]), "action": action})
            return action

        return choose
