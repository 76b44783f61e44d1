"""Whole lookahead_schedule of a config on one GPU: decisions, candidates,
wall time, makespan (development / demonstration aid)."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import instance  # noqa: E402
from paper_2604_23838_b200 import drive, simulate  # noqa: E402
from paper_2604_23838_b200.native import Evaluator  # noqa: E402

cfg, window = sys.argv[1], int(sys.argv[2])
cap = None if sys.argv[3] == "none" else int(sys.argv[3])
inst = instance(cfg)
ev = Evaluator(inst)
log = []
lat = []
choose = ev.chooser(window, cap, log)


def timed(state):
    t = time.perf_counter()
    a = choose(state)
    lat.append(time.perf_counter() - t)
    return a


t0 = time.perf_counter()
s = drive(inst, timed, "lookahead", {})
wall = time.perf_counter() - t0
rep = simulate(s, inst)
n = [d["n"] for d in log]
print(json.dumps({"config": cfg, "window": window, "max_merge": cap, "decisions": len(lat), "actions": len(s.actions),
                  "candidates_total": sum(n), "max_candidates": max(n), "wall_s": wall,
                  "p50_decision_ms": sorted(lat)[len(lat) // 2] * 1e3, "makespan": rep.makespan,
                  "throughput": rep.aggregate_throughput}))
