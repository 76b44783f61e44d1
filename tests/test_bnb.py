"""Brute-force oracle as native branch-and-bound (
rlmux/scheduler.py:1086-1226) and the serial policy (:983-1006).

tests/golden/bnb.json.gz holds the live reference's brute_force_schedule
and serial_schedule results on every committed fixture with <= 10
sub-stages (tests/golden/make_bnb_golden.py). CPU: the native search,
seeded with the CPU oracle's look-ahead / greedy schedules (the device
seeds need a GPU), returns the reference's schedule action for action.
GPU: the same with the device seeds (the product path).
"""
import pytest

from helpers import fixtures, load_gz


@pytest.fixture(scope="module")
def golden():
    return load_gz("bnb.json.gz")


def _json(sched):
    from paper_2604_23838_b200.instance_io import action_from, action_to_json

    return [[t.start, action_to_json(action_from(t.action))] for t in sched.actions]


def _oracle_seeds(inst):
    from oracle.oracle import Oracle
    from paper_2604_23838_b200 import drive
    from paper_2604_23838_b200.scheduler import serial_schedule

    o = Oracle(inst, nthreads=1)
    return [lambda i: drive(i, o.chooser(3), "lookahead", {}), lambda i: drive(i, o.chooser(1), "greedy", {}),
            serial_schedule]


def test_serial_schedule_matches_reference(golden):
    from paper_2604_23838_b200.scheduler import serial_schedule

    fx = fixtures()
    for name, rec in sorted(golden.items()):
        want = rec["serial"]
        if "raises" in want:
            continue
        assert _json(serial_schedule(fx[name])) == want["actions"], name


def test_branch_and_bound_matches_reference_cpu_seeds(golden):
    from paper_2604_23838_b200.model import OracleLimitError
    from paper_2604_23838_b200.scheduler import brute_force_schedule
    from paper_2604_23838_b200.sim import simulate

    fx = fixtures()
    checked = 0
    for name, rec in sorted(golden.items()):
        want = rec["oracle"]
        inst = fx[name]
        got = brute_force_schedule(inst, _seeds=_oracle_seeds(inst))
        assert _json(got) == want["actions"], name
        assert simulate(got, inst).makespan == want["makespan"], name
        assert got.metadata == want["metadata"], name
        checked += 1
    assert checked >= 100
    with pytest.raises(OracleLimitError, match="above the limit of 10"):
        from helpers import instance

        brute_force_schedule(instance("config1"))


@pytest.mark.gpu
def test_branch_and_bound_matches_reference_device_seeds(golden):
    from paper_2604_23838_b200.scheduler import brute_force_schedule

    fx = fixtures()
    for name in ("trap",) + tuple(sorted(n for n in golden if n.startswith("rand")))[:40]:
        assert _json(brute_force_schedule(fx[name])) == golden[name]["oracle"]["actions"], name
