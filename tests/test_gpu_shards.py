"""Cost-balanced multi-GPU parts on one GPU.

Each rank of an N-GPU decision scores part `rank` of `N` (RLX_F_SHARD: every
N-th block of 32 serials of each candidate class). Scoring the N parts one
after another on one device must
  * cover every candidate exactly once (candidate counts add up),
  * give the single-GPU winner as the lexicographic min of the part winners,
  * split the work evenly: max/mean of the parts' list-scheduling passes
    <= 1.10 (passes are deterministic; tools/shard_balance.py records the
    kernel-time ratio on hardware, profiles/r02_shard_balance_*.json).
"""
import statistics

import pytest

from helpers import instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,window,cap", [("config2", 2, None), ("config3", 3, 3), ("config4", 3, 2),
                                            ("config5", 4, 2)])
@pytest.mark.parametrize("n", [2, 8])
def test_parts_cover_balance_and_agree(Evaluator, cfg, window, cap, n):
    from paper_2604_23838_b200.state import State

    inst = instance(cfg)
    ev = Evaluator(inst)
    st = State(inst)
    whole = ev.decide(st, window, cap)
    parts = [ev.decide(st, window, cap, part=(r, n)) for r in range(n)]
    assert sum(p.passes for p in parts) == whole.passes
    best = min((p.cost, p.finish, p.priority, p.serial) for p in parts if p.found)
    assert best == (whole.cost, whole.finish, whole.priority, whole.serial)
    ps = [p.passes for p in parts]
    assert max(ps) / statistics.mean(ps) <= 1.10, ps
