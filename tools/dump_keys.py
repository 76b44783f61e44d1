"""Dump every device key (cost, finish) of a first decision (development aid:
input to tests/golden/make_sampled_keys.py, which picks the candidates the
oracle re-scores in the build container).

    python tools/dump_keys.py <config> <window> <cap|none> <out.npz>
"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import instance  # noqa: E402
from paper_2604_23838_b200.native import Evaluator  # noqa: E402
from paper_2604_23838_b200.state import State  # noqa: E402

cfg, w = sys.argv[1], int(sys.argv[2])
cap = None if sys.argv[3] == "none" else int(sys.argv[3])
inst = instance(cfg)
ev = Evaluator(inst)
st = State(inst)
d = ev.decide(st, w, cap, shard=(0, -1), want_keys=True)
np.savez_compressed(sys.argv[4], keys=ev.keys, winner=np.array([d.cost, d.finish, d.priority, d.serial]),
                    counts=np.array([d.n_multiplex, d.n_merge, d.n_exclusive]))
print(cfg, d.n_candidates, (d.cost, d.finish, d.priority, d.serial), d.kernel_ms)
