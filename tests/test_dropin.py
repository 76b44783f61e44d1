"""Drop-in boundary on CPU: rlmux objects in, rlmux objects out.

Builds instances with the live reference (/root/reference, build container
only; skipped elsewhere), converts them with `instance_io.as_instance`,
drives this package's decision loop with the oracle chooser (the device
chooser needs a GPU), converts the schedule back to rlmux's action classes
and replays it with the reference's own `rlmux.sim.simulate`: the result must
equal the reference's `lookahead_schedule` action for action."""

import inspect
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture(scope="module")
def rlmux():
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rlmux.fixtures
    import rlmux.scheduler
    import rlmux.sim

    return rlmux


def _reference_instances(rlmux):
    yield "trap", rlmux.fixtures.lookahead_trap_instance()
    for s in (3, 17, 42):
        yield f"rand{s}", rlmux.fixtures.random_small_instance(s)


@pytest.mark.parametrize("window", [1, 3])
def test_oracle_loop_on_reference_objects(rlmux, window):
    from oracle.oracle import Oracle
    from paper_2604_23838_b200 import drive
    from paper_2604_23838_b200.instance_io import action_as, as_instance

    for name, ref_inst in _reference_instances(rlmux):
        inst = as_instance(ref_inst)
        mine = drive(inst, Oracle(inst, nthreads=2).chooser(window), "lookahead", {})
        theirs = rlmux.scheduler.lookahead_schedule(ref_inst, window=window)
        conv = rlmux.scheduler.Schedule(
            actions=[rlmux.scheduler.TimedAction(t.start, action_as(t.action, rlmux.scheduler)) for t in mine.actions],
            policy="lookahead", metadata={})
        assert [(t.start, t.action) for t in conv.actions] == [(t.start, t.action) for t in theirs.actions], name
        a = rlmux.sim.simulate(conv, ref_inst)
        b = rlmux.sim.simulate(theirs, ref_inst)
        assert (a.makespan, a.aggregate_throughput) == (b.makespan, b.aggregate_throughput), name


def test_entry_point_signatures_match(rlmux):
    from paper_2604_23838_b200 import greedy_schedule, lookahead_schedule

    for ours, theirs in ((lookahead_schedule, rlmux.scheduler.lookahead_schedule),
                         (greedy_schedule, rlmux.scheduler.greedy_schedule)):
        po = inspect.signature(ours).parameters
        pt = inspect.signature(theirs).parameters
        for n, p in pt.items():
            assert n in po, n
            assert po[n].default == p.default, n
