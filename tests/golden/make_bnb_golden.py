"""Golden brute-force (and serial) schedules from the live reference.

TEST INFRASTRUCTURE ONLY (build container): runs rlmux's own
`brute_force_schedule` (scheduler.py:1148-1218) and `serial_schedule`
(:983-1006) on the committed trap and random fixtures with at most 10
sub-stages and writes tests/golden/bnb.json.gz (actions, makespan).

    python tests/golden/make_bnb_golden.py
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True


def main():
    import rlmux.scheduler as rs
    import rlmux.sim as rsim

    from helpers import fixtures
    from paper_2604_23838_b200.instance_io import action_from, action_to_json, to_reference

    out = {}
    for name, inst in sorted(fixtures().items()):
        if sum(len(g.nodes) for g in inst.graphs) > 10:
            continue
        ri = to_reference(inst)
        rec = {}
        for pol, fn in (("oracle", rs.brute_force_schedule), ("serial", rs.serial_schedule)):
            t = time.time()
            try:
                s = fn(ri)
            except Exception as exc:  # noqa: BLE001 - recorded as the reference's outcome
                rec[pol] = {"raises": type(exc).__name__, "message": str(exc)}
                continue
            rec[pol] = {"actions": [[a.start, action_to_json(action_from(a.action))] for a in s.actions],
                        "makespan": rsim.simulate(s, ri).makespan, "metadata": dict(s.metadata),
                        "secs": time.time() - t}
        out[name] = rec
    path = os.path.join(HERE, "bnb.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(out, fh)
    print("wrote", path, len(out), "instances")


if __name__ == "__main__":
    main()
