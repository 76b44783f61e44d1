"""Batched replay of schedules (rlmux/sim.py:69-173):
`simulate_batch` (native, all host threads, csrc/rlx_sim.cpp) gives the same
metrics as `simulate` for every golden schedule, bit for bit, and the
makespan / throughput the live reference recorded."""
import pytest

from helpers import instance


def _schedules(golden, names):
    from paper_2604_23838_b200.instance_io import action_from_json
    from paper_2604_23838_b200.model import Schedule, TimedAction

    out = {}
    for n in names:
        g = golden[n]
        out.setdefault(g["instance"], []).append(
            (n, g, Schedule(actions=[TimedAction(t, action_from_json(a)) for t, a in g["actions"]],
                            policy="lookahead", metadata={})))
    return out


def test_batch_equals_single_replay(golden_schedules):
    from paper_2604_23838_b200.sim import simulate, simulate_batch

    names = sorted(golden_schedules)
    by_inst = _schedules(golden_schedules, names)
    checked = 0
    for iname, rows in by_inst.items():
        inst = instance(iname)
        reps = simulate_batch([s for _, _, s in rows], inst, threads=4)
        for (n, g, s), r in zip(rows, reps):
            one = simulate(s, inst)
            assert (r.makespan, r.aggregate_throughput) == (g["makespan"], g["throughput"]), n
            assert r.makespan == one.makespan and r.aggregate_throughput == one.aggregate_throughput, n
            assert r.per_pipeline_latency == one.per_pipeline_latency, n
            assert list(r.per_pipeline_latency) == list(one.per_pipeline_latency), n
            assert r.per_pipeline_tokens == one.per_pipeline_tokens, n
            assert r.utilization_avg == one.utilization_avg, n
            checked += 1
    assert checked == len(names)


def test_batch_reports_dependency_violations():
    from paper_2604_23838_b200.model import Exclusive, Schedule, TimedAction
    from paper_2604_23838_b200.sim import DependencyViolationError, simulate, simulate_batch

    inst = instance("trap")
    bad = Schedule(actions=[TimedAction(0.0, Exclusive("no/such/node"))], policy="x", metadata={})
    with pytest.raises(DependencyViolationError) as e1:
        simulate(bad, inst)
    with pytest.raises(DependencyViolationError) as e2:
        simulate_batch([bad], inst)
    assert str(e1.value) == str(e2.value)
    empty = Schedule(actions=[], policy="x", metadata={})
    with pytest.raises(DependencyViolationError) as e3:
        simulate(empty, inst)
    with pytest.raises(DependencyViolationError) as e4:
        simulate_batch([empty], inst)
    assert str(e3.value) == str(e4.value)


def test_utilization_matches_live_reference(golden_schedules):
    """Our utilisation fold (sim.py) and the batch's equal the reference's
    `_utilization` (rlmux/sim.py:69-115) on rlmux objects (build container
    only)."""
    import os
    import sys

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.dont_write_bytecode = True
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import rlmux.scheduler as rs
    import rlmux.sim as rsim

    from paper_2604_23838_b200.instance_io import action_as, action_from_json, to_reference
    from paper_2604_23838_b200.model import Schedule, TimedAction
    from paper_2604_23838_b200.sim import simulate, simulate_batch

    for name in ("trap_w3", "config1_w1", "async_small_w3_cap3", "rand012_w3", "rand031_w1"):
        g = golden_schedules[name]
        inst = instance(g["instance"])
        ours = Schedule(actions=[TimedAction(t, action_from_json(a)) for t, a in g["actions"]], policy="lookahead",
                        metadata={})
        rinst = to_reference(inst)
        theirs = rs.Schedule(actions=[rs.TimedAction(t.start, action_as(t.action, rs)) for t in ours.actions],
                             policy="lookahead", metadata={})
        want = rsim.simulate(theirs, rinst)
        one = simulate(ours, inst)
        batch = simulate_batch([ours], inst)[0]
        assert one.utilization_avg == want.utilization_avg == batch.utilization_avg, name
        assert one.utilization_series == want.utilization_series, name
        assert [(e.time, e.worker_id, e.kind, e.node_id, e.alloc) for e in one.events] == [
            (e.time, e.worker_id, e.kind, e.node_id, e.alloc) for e in want.events], name
