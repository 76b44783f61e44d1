"""One warm-up + one measured decision at a config (ncu target).

    python tools/ncu_target.py <config> <window> <cap|none> [n_serials | begin:end]
"""
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import instance  # noqa: E402
from paper_2604_23838_b200.state import State as HostState  # noqa: E402
from paper_2604_23838_b200.native import Evaluator  # noqa: E402

cfg = sys.argv[1]
w = int(sys.argv[2])
cap = None if sys.argv[3] == "none" else int(sys.argv[3])
shard = None
if len(sys.argv) > 4:
    a = sys.argv[4]
    shard = tuple(int(x) for x in a.split(":")) if ":" in a else (0, int(a))
inst = instance(cfg)
ev = Evaluator(inst)
st = HostState(inst)
for _ in range(2):
    d = ev.decide(st, w, cap, shard=shard)
print(cfg, d.n_candidates, d.kernel_ms, d.passes, d.alg_bytes)
