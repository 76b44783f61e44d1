"""Development aid: score sampled golden candidates under forced lane shapes
(needs librlx_dbg.so, RLX_LIB pointing at it)."""
import os
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import instance, load_gz  # noqa: E402
from paper_2604_23838_b200.engine import HostState  # noqa: E402
from paper_2604_23838_b200.native import Evaluator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config3"
g = load_gz("keys.json.gz")[name]
inst = instance(g["instance"])
st = HostState(inst)
ev = Evaluator(inst)
for shape in ["32,1", "16,2", "8,4", "4,8"]:
    os.environ["RLX_SHAPE"] = shape
    bad = 0
    for serial, prio, cost, fin in g["keys"][:8]:
        ev.decide(st, g["window"], g["max_merge"], shard=(serial, serial + 1), want_keys=True)
        got = tuple(ev.keys[0])
        if got != (cost, fin):
            bad += 1
            print(shape, serial, "got", got, "want", (cost, fin), flush=True)
    print("shape", shape, "bad", bad, flush=True)
