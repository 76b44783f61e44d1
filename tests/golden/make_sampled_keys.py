"""Oracle keys for a stratified sample of the config-5 (merge cap 2) first
decision — the bench headline, too large to score completely on the CPU
(~12 h on 16 threads).

TEST INFRASTRUCTURE ONLY. Input: the device's full key dump of the decision
(`python tools/dump_keys.py config5 4 2 gpurun_out/keys_config5_cap2.npz`
on a GPU box). The sample is
  * every candidate whose device cost equals the device winner's cost
    (the ties the (finish, priority, serial) tie-break decides), and
  * a class-stratified uniform sample (multiplex, merge, exclusive),
scored here by the CPU oracle (pinned to the live reference by
tests/test_oracle.py). Writes tests/golden/full/config5_cap2_sample.npz:
serials, oracle keys, classes, and the winner — the device winner, kept
only if the oracle reproduces its key and no sampled candidate beats it.

    python tests/golden/make_sampled_keys.py gpurun_out/keys_config5_cap2.npz
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

PER_CLASS = {"multiplex": 200, "merge": 260, "exclusive": 48}


def main(dump: str, seed: int = 2) -> None:
    from helpers import instance
    from oracle.oracle import Oracle
    from paper_2604_23838_b200.state import State

    dev = np.load(dump)
    keys, winner = dev["keys"], dev["winner"]
    n_mux, n_merge, n_excl = (int(x) for x in dev["counts"])
    n = n_mux + n_merge + n_excl
    assert keys.shape[0] == n
    rng = np.random.default_rng(seed)
    ties = np.nonzero(keys[:, 0] == winner[0])[0]
    picks = [ties]
    for name, (lo, hi) in {"multiplex": (0, n_mux), "merge": (n_mux, n_mux + n_merge),
                           "exclusive": (n_mux + n_merge, n)}.items():
        k = min(PER_CLASS[name], hi - lo)
        picks.append(lo + rng.choice(hi - lo, size=k, replace=False))
    serials = np.unique(np.concatenate(picks + [np.array([int(winner[3])])]))
    prio = np.where(serials < n_mux, 0, np.where(serials < n_mux + n_merge, 1, 2)).astype(np.uint8)
    print(f"{serials.size} serials ({ties.size} cost ties with the winner)", flush=True)
    inst = instance("config5")
    st = State(inst)
    o = Oracle(inst, nthreads=os.cpu_count())
    t = time.time()
    r = o.score(st, 4, 2, serials=serials, want_keys=True)
    print(f"oracle scored them in {time.time() - t:.0f} s", flush=True)
    ok = r["keys"]
    agree = (ok.view(np.uint64) == keys[serials].view(np.uint64)).all(axis=1)
    print(f"device == oracle on {int(agree.sum())}/{serials.size}", flush=True)
    wkey = (float(winner[0]), float(winner[1]), int(winner[2]), int(winner[3]))
    for s, (c, f), p in zip(serials, ok, prio):
        assert wkey <= (c, f, int(p), int(s)), (s, c, f, p)
    i = int(np.searchsorted(serials, wkey[3]))
    assert (ok[i, 0], ok[i, 1]) == wkey[:2]
    out = os.path.join(HERE, "full", "config5_cap2_sample.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(out, serials=serials, keys=ok, prio=prio, winner=np.array(wkey, dtype=np.float64),
                        counts=np.array([n_mux, n_merge, n_excl]))
    print("wrote", out, os.path.getsize(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
