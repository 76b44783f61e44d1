"""Confirm on the live reference that a first-decision candidate livelocks
(raises SchedulingError at the 10,000-advance guard, scheduler.py:866).

TEST INFRASTRUCTURE ONLY (needs /root/reference; build container).

    python tests/golden/check_livelock.py config5 4 3 819010

Appends {"<cfg>:<serial>": {"raises": bool, "message": str, "seconds": s}}
to tests/golden/livelock.json.
"""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import refharness as H  # noqa: E402
from make_golden import _load_fixture  # noqa: E402
from rlmux.scheduler import SchedulingError  # noqa: E402


def main():
    cfg, window, cap, serial = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    inst = _load_fixture(cfg)
    st = H.ExecState(inst)
    t = time.time()
    with H.capped(cap):
        cands = H.capped_enumerate(st, cap)
        cand = cands[serial]
        assert cand.serial == serial
        try:
            H.candidate_cost(st, cand.action, window)
            res = {"raises": False, "message": ""}
        except SchedulingError as e:
            res = {"raises": True, "message": str(e)}
    res["seconds"] = time.time() - t
    res["action"] = H.action_to_json(cand.action)
    path = os.path.join(HERE, "livelock.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out[f"{cfg}:{serial}"] = res
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(cfg, serial, res)


if __name__ == "__main__":
    main()
