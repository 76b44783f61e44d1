"""The product kernel source, compiled for the host as a one-lane debugging
twin (tests/twin), replays golden schedules and candidate keys of the
reference bit-exactly on CPU. This checks the event-loop logic of
paper_2604_23838_b200/csrc/rlx_kernels.cu without a GPU; the device itself
is checked in test_gpu_parity.py."""

import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "twin"))

from helpers import instance  # noqa: E402
from paper_2604_23838_b200 import drive  # noqa: E402
from paper_2604_23838_b200.state import State as HostState  # noqa: E402
from paper_2604_23838_b200.instance_io import action_to_json  # noqa: E402


@pytest.fixture(scope="module", params=["lean", "u"])
def Twin(request):
    """The twin class bound to one consume variant (twin/Makefile)."""
    import functools
    import shutil

    if shutil.which(os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")) is None and not os.path.exists(
            "/usr/local/cuda/bin/nvcc"):
        pytest.skip("nvcc not available")
    from twin import Twin as T

    return functools.partial(T, variant=request.param)


def _twin_chooser(Twin, inst, window, cap, log):
    import numpy as np

    from oracle.oracle import Oracle

    t = Twin(inst)
    o = Oracle(inst, nthreads=1)

    def choose(state):
        rc, err, n, key, dbg, keys = t.decide(state, window, cap, shard=(0, -1))
        assert rc == 0, err
        if n == 0:
            return None
        k = np.array(key[:3], dtype=np.uint64)
        cost, fin = (float(x) for x in k[:2].view(np.float64))
        prio, serial = int(k[2]) >> 61, int(k[2]) & ((1 << 61) - 1)
        log.append({"n": n, "key": [cost, fin, prio, serial]})
        return o.candidate(state, serial, cap)

    return choose


def test_twin_golden_schedules(Twin, golden_schedules):
    names = sorted(golden_schedules)
    picked = [n for n in names if not n.startswith("rand")] + [n for n in names if n.startswith("rand")][::7]
    bad = []
    for name in picked:
        g = golden_schedules[name]
        inst = instance(g["instance"])
        if len(inst.workers()) > 32:
            continue
        log = []
        s = drive(inst, _twin_chooser(Twin, inst, g["window"], g["max_merge"], log), "lookahead", {})
        acts = [[t.start, action_to_json(t.action)] for t in s.actions]
        keys_ok = len(log) == len(g["decisions"]) and all(
            d["n"] == gd["n"] and list(d["key"]) == list(gd["key"]) for d, gd in zip(log, g["decisions"]))
        if acts != g["actions"] or not keys_ok:
            bad.append(name)
    assert not bad, bad[:6]


def test_twin_golden_schedules_knobs(Twin, golden_schedules_knobs):
    bad = []
    for name in sorted(golden_schedules_knobs)[::3]:
        g = golden_schedules_knobs[name]
        inst = instance(g["instance"])
        log = []
        s = drive(inst, _twin_chooser(Twin, inst, g["window"], g["max_merge"], log), "lookahead", {})
        acts = [[t.start, action_to_json(t.action)] for t in s.actions]
        if acts != g["actions"] or [d["key"] for d in log] != [list(d["key"]) for d in g["decisions"]]:
            bad.append(name)
    assert not bad, bad[:6]


@pytest.mark.parametrize("name", ["trap", "async_small", "config1", "config2", "config3"])
def test_twin_candidate_keys(Twin, golden_keys, name):
    g = golden_keys[name]
    inst = instance(g["instance"])
    st = HostState(inst)
    t = Twin(inst)
    for serial, prio, cost, fin in g["keys"][:16]:
        rc, err, n, key, dbg, keys = t.decide(st, g["window"], g["max_merge"], shard=(serial, serial + 1))
        assert rc == 0, err
        assert n == g["n_candidates"]
        assert tuple(keys[0]) == (cost, fin), (name, serial)
