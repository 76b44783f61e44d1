"""Every key of the benchmarked decisions, bit-exact against golden data.

tests/golden/full/<name>.keys.xz holds the CPU oracle's (cost, finish) for
EVERY candidate of a first decision and <name>.npz the (cost, finish,
priority, serial) winner (tests/golden/make_full_keys.py; the oracle is pinned to the live
reference by tests/test_oracle.py). tests/golden/full/<name>_sample.npz
holds oracle keys for a stratified sample of a decision too large to score
completely on the CPU (config 5, merge cap 2: every candidate tied with the
device winner on cost, plus a class-stratified sample;
tests/golden/make_sampled_keys.py).

The device scores the whole decision through the C-ABI (rlx_decide with a
keys buffer) and must reproduce all of them and the winner exactly
(tolerance 0; the north star allows 1e-9 relative).
"""
import os

import numpy as np
import pytest

from helpers import GOLDEN, instance

FULL = os.path.join(GOLDEN, "full")
JOBS = {
    # name: (instance, window, max_merge)
    "config2_full": ("config2", 2, None),
    "config4_cap2": ("config4", 3, 2),
    "config3_cap3": ("config3", 3, 3),
    "config5_cap2": ("config5", 4, 2),
}


def _have(name):
    return os.path.exists(os.path.join(FULL, f"{name}.npz")) and os.path.exists(os.path.join(FULL, f"{name}.keys.xz"))


def _keys(name):
    """(cost, finish) of every serial: raw little-endian float64, lzma."""
    import lzma

    with lzma.open(os.path.join(FULL, f"{name}.keys.xz"), "rb") as fh:
        return np.frombuffer(fh.read(), dtype="<f8").reshape(-1, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in JOBS if n != "config5_cap2"])
def test_full_decision_keys(Evaluator, name):
    if not _have(name):
        pytest.skip(f"golden {name} not generated")
    from paper_2604_23838_b200.state import State

    g = np.load(os.path.join(FULL, f"{name}.npz"))
    keys = _keys(name)
    cfg, window, cap = JOBS[name]
    inst = instance(cfg)
    ev = Evaluator(inst)
    st = State(inst)
    d = ev.decide(st, window, cap, shard=(0, -1), want_keys=True)
    n = keys.shape[0]
    assert d.n_candidates == n
    assert (d.n_multiplex, d.n_merge, d.n_exclusive) == (int(g["n_mux"]), int(g["n_merge"]), int(g["n_excl"]))
    got = ev.keys.view(np.uint64)
    want = keys.view(np.uint64)
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} of {n} keys differ, first serials {bad[:8].tolist()}"
    assert (d.cost, d.finish, d.priority, d.serial) == tuple(
        float(x) if i < 2 else int(x) for i, x in enumerate(g["winner"]))
    # the plain decision (no keys buffer) picks the same winner
    d2 = ev.decide(st, window, cap)
    assert (d2.cost, d2.finish, d2.priority, d2.serial) == (d.cost, d.finish, d.priority, d.serial)


@pytest.mark.gpu
def test_config5_cap2_sampled_keys(Evaluator):
    """Config 5 (merge cap 2), the bench headline: every candidate whose cost
    equals the winner's, plus a class-stratified sample, keyed by the
    oracle; the device's full decision must match all of them, and no
    sampled candidate may beat the device winner."""
    path = os.path.join(FULL, "config5_cap2_sample.npz")
    if not os.path.exists(path):
        pytest.skip("golden config5_cap2_sample not generated")
    from paper_2604_23838_b200.state import State

    g = np.load(path)
    inst = instance("config5")
    ev = Evaluator(inst)
    st = State(inst)
    d = ev.decide(st, 4, 2, shard=(0, -1), want_keys=True)
    serials = g["serials"]
    got = ev.keys[serials].view(np.uint64)
    want = g["keys"].view(np.uint64)
    bad = serials[(got != want).any(axis=1)]
    assert bad.size == 0, f"{bad.size} of {serials.size} sampled keys differ: {bad[:8].tolist()}"
    assert (d.cost, d.finish, d.priority, d.serial) == tuple(
        float(x) if i < 2 else int(x) for i, x in enumerate(g["winner"]))
    prio = g["prio"]
    for s, (c, f), p in zip(serials, g["keys"], prio):
        assert (d.cost, d.finish, d.priority, d.serial) <= (c, f, int(p), int(s))
