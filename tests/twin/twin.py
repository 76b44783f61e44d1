"""ctypes front-end of the host debugging twin (test infrastructure only)."""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2604_23838_b200 import abi
from paper_2604_23838_b200.encode import instance_encoding

HERE = os.path.dirname(os.path.abspath(__file__))
# "lean": the lane split of >= 16-lane device groups; "u": consume_u (smaller groups)
LIBS = {"lean": os.path.join(HERE, "_build", "librlx_twin.so"), "u": os.path.join(HERE, "_build", "librlx_twin_u.so")}
VARIANT = os.environ.get("RLX_TWIN_VARIANT", "lean")
_libs = {}


def lib(variant=None):
    variant = variant or VARIANT
    if variant not in _libs:
        subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = C.CDLL(LIBS[variant])
        L.rlx_twin_decide.restype = C.c_int
        L.rlx_twin_decide.argtypes = [C.POINTER(abi.RlxInstanceDesc), C.POINTER(abi.RlxStateDesc), C.c_int, C.c_int,
                                      C.c_int64, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.c_char_p, C.c_int]
        _libs[variant] = L
    return _libs[variant]


class Twin:
    def __init__(self, instance, variant=None):
        self.enc = instance_encoding(instance)
        self.variant = variant

    def decide(self, state, window, max_merge=None, shard=(0, -1), want_keys=True):
        sd = state.snapshot()
        n = C.c_int64()
        key = (C.c_uint64 * 4)()
        dbg = (C.c_double * 16)()
        err = C.create_string_buffer(256)
        b, e = shard
        keys = np.zeros((max(1, (e - b) if e >= 0 else 4_000_000), 2))
        rc = lib(self.variant).rlx_twin_decide(C.byref(self.enc.desc), C.byref(sd), window, 0 if max_merge is None else max_merge,
                                   b, e, keys.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n), key, dbg, err, 256)
        return rc, err.value.decode(), n.value, list(key), list(dbg), keys
