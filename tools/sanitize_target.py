"""Small decisions for compute-sanitizer (memcheck / racecheck / synccheck):
the trap fixture at W=3, a config-2 cap-3 shard, a config-3 shard and a
config-4 shard with tool waits."""
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import instance  # noqa: E402
from paper_2604_23838_b200.state import State as HostState  # noqa: E402
from paper_2604_23838_b200.native import Evaluator  # noqa: E402

for name, w, cap, shard in (("trap", 3, None, None), ("config2", 2, 3, (0, 400)), ("config3", 3, 3, (8000, 8100)),
                            ("config4", 3, 3, (0, 40))):
    inst = instance(name)
    ev = Evaluator(inst)
    d = ev.decide(HostState(inst), w, cap, shard=shard)
    print(name, d.n_candidates, d.cost, d.serial, flush=True)
