"""Drop-in on the GPU: the reference's own objects through the device
`lookahead_schedule`.

The unmodified reference (rlmux, installed into baseline/_ref from
/root/reference; skipped when absent) gets instances built from the
committed golden JSON (`instance_io.to_reference`). Those rlmux Instances go
through this package's `lookahead_schedule` (device chooser, native decision
loop); the returned rlmux Schedule must equal the committed live-reference
schedule action for action, and the reference's own `rlmux.sim.simulate`
must give the committed makespan and throughput.
"""
import os
import sys

import pytest

from helpers import ROOT, instance

REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "rlmux")), reason="baseline/_ref not installed")]

CASES = ["trap_w1", "trap_w3", "config1_w1", "config1_w3", "async_small_w3_cap3", "rand007_w3", "rand042_w1"]


@pytest.fixture(scope="module")
def rlmux():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rlmux.scheduler
    import rlmux.sim

    return rlmux


@pytest.mark.parametrize("name", CASES)
def test_reference_objects_through_device(rlmux, golden_schedules, name):
    from paper_2604_23838_b200 import lookahead_schedule
    from paper_2604_23838_b200.instance_io import action_from_json, action_to_json, action_from, to_reference

    if name not in golden_schedules:
        pytest.skip(f"{name} not in the golden set")
    g = golden_schedules[name]
    ref_inst = to_reference(instance(g["instance"]))
    sched = lookahead_schedule(ref_inst, window=int(g["window"]), max_merge=g["max_merge"])
    assert type(sched).__module__.startswith("rlmux")
    got = [[t.start, action_to_json(action_from(t.action))] for t in sched.actions]
    want = [[t, action_to_json(action_from_json(a))] for t, a in g["actions"]]
    assert got == want
    rep = rlmux.sim.simulate(sched, ref_inst)
    assert (rep.makespan, rep.aggregate_throughput) == (g["makespan"], g["throughput"])
