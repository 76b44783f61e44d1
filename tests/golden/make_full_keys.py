"""Full-decision oracle scorings of the benchmarked decisions (golden data).

TEST INFRASTRUCTURE ONLY. Scores EVERY candidate of a first decision with
the CPU oracle (oracle/rlx_oracle.c, pinned to the live reference by
tests/test_oracle.py) on all host threads, and writes

    tests/golden/full/<name>.keys.xz   float64 [n, 2] (cost, finish) per serial,
                                       little-endian, lzma-compressed
    tests/golden/full/<name>.npz       winner float64 [4] (cost, finish,
                                       priority, serial) argmin; n_mux,
                                       n_merge, n_excl; window; max_merge

so the GPU parity tests can compare every device key and the winner
bit-exactly (tests/test_gpu_full_decisions.py). Run in the build container
(no GPU needed); resumable: finished chunks are kept under /tmp.

    python tests/golden/make_full_keys.py config2_full      # W=2, uncapped, 1,048,864 candidates
    python tests/golden/make_full_keys.py config4_cap2      # W=3, cap 2, 23,296 candidates
    python tests/golden/make_full_keys.py config3_cap3      # W=3, cap 3, 71,808 candidates
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

JOBS = {
    # name: (instance, window, max_merge)
    "config2_full": ("config2", 2, None),
    "config4_cap2": ("config4", 3, 2),
    "config3_cap3": ("config3", 3, 3),
    "config5_cap2": ("config5", 4, 2),
}
CHUNK = 1 << 14


def main(name: str, threads: int | None = None) -> None:
    from helpers import instance
    from oracle.oracle import Oracle
    from paper_2604_23838_b200.state import State

    inst_name, window, cap = JOBS[name]
    inst = instance(inst_name)
    st = State(inst)
    o = Oracle(inst, nthreads=threads or os.cpu_count())
    n = o.score(st, window, cap, serials=[])["n"]
    tmp = f"/tmp/full_keys_{name}"
    os.makedirs(tmp, exist_ok=True)
    keys = np.zeros((n, 2), dtype=np.float64)
    t0 = time.time()
    for b in range(0, n, CHUNK):
        e = min(n, b + CHUNK)
        path = os.path.join(tmp, f"{b:09d}.npy")
        if os.path.exists(path):
            keys[b:e] = np.load(path)
            continue
        r = o.score(st, window, cap, serials=np.arange(b, e), want_keys=True)
        keys[b:e] = r["keys"]
        np.save(path, r["keys"])
        done = e
        print(f"{name}: {done}/{n} in {time.time() - t0:.0f}s", flush=True)
    # candidate classes from the serial layout (multiplex, merges, exclusives)
    prio = np.zeros(n, dtype=np.uint8)
    n_mux, n_merge, _ = o.counts(st, window, cap)
    prio[n_mux:n_mux + n_merge] = 1
    prio[n_mux + n_merge:] = 2
    order = np.lexsort((np.arange(n), prio, keys[:, 1], keys[:, 0]))
    w = int(order[0])
    winner = np.array([keys[w, 0], keys[w, 1], prio[w], w], dtype=np.float64)
    os.makedirs(os.path.join(HERE, "full"), exist_ok=True)
    out = os.path.join(HERE, "full", f"{name}.npz")
    save_keys(os.path.join(HERE, "full", f"{name}.keys.xz"), keys)
    np.savez_compressed(out, winner=winner, n_mux=n_mux, n_merge=n_merge,
                        n_excl=n - n_mux - n_merge, window=window, max_merge=-1 if cap is None else cap)
    print("wrote", out, os.path.getsize(out), "winner", winner.tolist(), flush=True)


def save_keys(path, keys):
    import lzma

    with lzma.open(path, "wb", preset=9) as fh:
        fh.write(np.ascontiguousarray(keys, dtype="<f8").tobytes())


def load_keys(path):
    import lzma

    with lzma.open(path, "rb") as fh:
        return np.frombuffer(fh.read(), dtype="<f8").reshape(-1, 2)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        main(nm)
