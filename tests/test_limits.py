"""The compiled limits of this build (include/rlx.h RLX_ERR_LIMIT,
INTEGRATION.md §4), probed with instances that cross each one.

The reference has no such limits; crossing one raises `CapacityError` with
the documented text from the host planner (`native.plan_info`, no GPU
needed) before any device work, instead of a wrong result. Just below each
limit the planner accepts the instance. Limits that cannot be reached
without crossing another first are noted where they are checked
(rlx_plan.cpp): the 60k-node window needs > 128 workers x 63 sub-stages.
"""
import pytest

from paper_2604_23838_b200.model import Instance, SubStage, SubStageGraph, SubStageKind, default_model
from paper_2604_23838_b200.native import CapacityError, plan_info
from paper_2604_23838_b200.state import State


def _inst(nodes_per_worker, n_workers, kind=SubStageKind.DECODE_SMALL, chains=False, pipelines=1):
    """`pipelines` graphs; on every worker `nodes_per_worker` independent
    sub-stages (or one chain of them), each with 1 active request."""
    graphs = []
    for p in range(pipelines):
        pid = f"p{p}"
        nodes, edges = {}, set()
        for w in range(n_workers):
            prev = None
            for i in range(nodes_per_worker):
                nid = f"{pid}/w{w}/n{i:03d}"
                nodes[nid] = SubStage(id=nid, pipeline_id=pid, worker_id=w, kind=kind, duration=1.0 + 0.01 * i,
                                      mem_fraction=0.3, remaining_decode_tokens=10, active_requests=1)
                if chains and prev is not None:
                    edges.add((prev, nid))
                prev = nid
        graphs.append(SubStageGraph(pid, nodes, edges, None, {0: 0.02, 1: 0.05, 2: 0.18}))
    return Instance(graphs=graphs, model=default_model())


def _plan(inst, window=1, max_merge=None):
    return plan_info(State(inst), window, max_merge)


def test_workers_128_ok_129_refused():
    assert _plan(_inst(1, 128, kind=SubStageKind.TRAINING)).n_candidates == 128
    with pytest.raises(CapacityError, match="more than 128 workers"):
        _plan(_inst(1, 129, kind=SubStageKind.TRAINING))


def test_window_substages_per_worker_63_ok_64_refused():
    assert _plan(_inst(63, 1, kind=SubStageKind.TRAINING)).max_worker_order == 63
    with pytest.raises(CapacityError, match="more than 63 window sub-stages on one worker"):
        _plan(_inst(64, 1, kind=SubStageKind.TRAINING))


def test_merge_set_size_64_ok_65_refused_unless_capped():
    # 65 ready DecodeSmall fragments of one pipeline on distinct workers:
    # the reference enumerates merge sets up to all 65 members
    with pytest.raises(CapacityError, match="merge sets above 64 members"):
        _plan(_inst(1, 65), max_merge=None)
    assert _plan(_inst(1, 65), max_merge=2).n_merge == 65 * 64  # C(65,2) pairs x 2 targets


def test_mergeable_fragments_per_pipeline_128_ok_129_refused():
    ok = _plan(_inst(2, 64), max_merge=2)  # 128 fragments on 64 workers
    assert ok.n_merge > 0
    with pytest.raises(CapacityError, match="more than 128 mergeable fragments"):
        _plan(_inst(3, 43), max_merge=2)  # 129 fragments


def test_shared_memory_plan_refused_with_text():
    # 128 workers x 63-sub-stage chains, W=63: ~8k window nodes do not fit the
    # 227 KB of shared memory a CTA stages the plan into
    with pytest.raises(CapacityError, match="does not fit in shared memory"):
        _plan(_inst(63, 128, kind=SubStageKind.TRAINING, chains=True), window=63)
