"""One-GPU emulation of the multi-GPU split: score parts
0..N-1 of a decision one after another (RLX_F_SHARD, the block-cyclic parts
each rank of an N-GPU run scores) and report each part's kernel time, passes
and simulated events, and max/mean — the speed-up ceiling of N GPUs is
N / (max/mean).

    python tools/shard_balance.py <config> <window> <cap|none> [N ...] > out.json
"""
import json
import statistics
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import instance  # noqa: E402
from paper_2604_23838_b200.native import Evaluator  # noqa: E402
from paper_2604_23838_b200.state import State  # noqa: E402

cfg, w = sys.argv[1], int(sys.argv[2])
cap = None if sys.argv[3] == "none" else int(sys.argv[3])
ns = [int(x) for x in sys.argv[4:]] or [2, 4, 8]
inst = instance(cfg)
ev = Evaluator(inst)
st = State(inst)
full = ev.decide(st, w, cap)
full = ev.decide(st, w, cap)  # warm
out = {"config": cfg, "window": w, "max_merge": cap, "candidates": full.n_candidates,
       "one_gpu_kernel_ms": full.kernel_ms, "winner": [full.cost, full.finish, full.priority, full.serial], "parts": {}}
for n in ns:
    rows = []
    for r in range(n):
        d = ev.decide(st, w, cap, part=(r, n))
        rows.append({"rank": r, "kernel_ms": d.kernel_ms, "passes": d.passes, "events": d.events,
                     "key": [d.cost, d.finish, d.priority, d.serial] if d.found else None})
    km = [x["kernel_ms"] for x in rows]
    ps = [x["passes"] for x in rows]
    best = min((tuple(x["key"]) for x in rows if x["key"]), default=None)
    out["parts"][str(n)] = {"ranks": rows, "kernel_max_over_mean": max(km) / statistics.mean(km),
                            "passes_max_over_mean": max(ps) / statistics.mean(ps),
                            "speedup_ceiling": n / (max(km) / statistics.mean(km)),
                            "sum_kernel_ms": sum(km), "winner_matches": list(best) == out["winner"]}
    print(f"{cfg} N={n}: kernel max/mean {max(km) / statistics.mean(km):.3f} passes max/mean "
          f"{max(ps) / statistics.mean(ps):.3f} winner ok {list(best) == out['winner']}", file=sys.stderr, flush=True)
print(json.dumps(out))
