"""Randomised cross-check of the kernel logic against the oracle (which is
pinned to the live reference by test_oracle.py): the golden fixture
instances under random Instance knobs, windows and merge caps; every
decision of the resulting schedule is scored by both, and the selected keys
must be bit-identical. CPU: the host twin of the kernel source. GPU: the
device through the C-ABI."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "twin"))

from helpers import fixtures  # noqa: E402
from paper_2604_23838_b200 import drive  # noqa: E402
from paper_2604_23838_b200.model import Instance  # noqa: E402


def cases(n, seed):
    rng = np.random.default_rng(seed)
    fx = fixtures()
    names = sorted(fx)
    for _ in range(n):
        base = fx[names[rng.integers(len(names))]]
        inst = Instance(graphs=base.graphs, model=base.model,
                        headroom=float(rng.choice([0.05, 0.1, 0.0, 0.2])),
                        realloc_penalty=float(rng.choice([0.0, 0.0, 0.3, 1.25])),
                        default_migration_cost=float(rng.choice([0.0, 0.1, 0.7])),
                        merge_enabled=bool(rng.random() < 0.85))
        window = int(rng.integers(1, 5))
        cap = [None, 2, 3][int(rng.integers(3))]
        yield inst, window, cap


def _compare(inst, window, cap, score_other):
    """Drive the schedule with the oracle; at every decision the other
    scorer must produce the same (n, best key)."""
    from oracle.oracle import Oracle

    o = Oracle(inst, nthreads=2)
    bad = []

    def choose(state):
        r = o.score(state, window, cap)
        other = score_other(state)
        if other != (r["n"], r["best"]):
            bad.append((state.now, other, (r["n"], r["best"])))
        if r["n"] == 0:
            return None
        return o.candidate(state, r["best"][3], cap)

    drive(inst, choose, "lookahead", {})
    return bad


def _key(rows):
    k = np.array(rows[:3], dtype=np.uint64)
    cost, fin = (float(x) for x in k[:2].view(np.float64))
    return cost, fin, int(k[2]) >> 61, int(k[2]) & ((1 << 61) - 1)


@pytest.mark.parametrize("variant", ["lean", "u"])
def test_twin_matches_oracle_on_random_knobs(variant):
    from twin import Twin

    failures = []
    for inst, window, cap in cases(40, seed=7):
        t = Twin(inst, variant=variant)

        def twin_score(state):
            rc, err, n, key, dbg, keys = t.decide(state, window, cap, shard=(0, -1))
            assert rc == 0, err
            return n, (None if n == 0 else _key(key))

        bad = _compare(inst, window, cap, twin_score)
        if bad:
            failures.append((window, cap, inst.headroom, inst.realloc_penalty, bad[0]))
    assert not failures, failures[:3]


@pytest.mark.gpu
def test_device_matches_oracle_on_random_knobs():
    from paper_2604_23838_b200.native import Evaluator

    failures = []
    ev = None
    for inst, window, cap in cases(80, seed=11):
        if ev is None:
            ev = Evaluator(inst)
        else:
            ev.bind(inst)

        def dev_score(state):
            d = ev.decide(state, window, cap)
            return d.n_candidates, (None if d.n_candidates == 0 else (d.cost, d.finish, d.priority, d.serial))

        bad = _compare(inst, window, cap, dev_score)
        if bad:
            failures.append((window, cap, inst.headroom, inst.realloc_penalty, bad[0]))
    assert not failures, failures[:3]
