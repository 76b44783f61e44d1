"""Multi-rank decision on CPU (gloo, world_size 2): each rank scores its
contiguous serial shard, packs its shard winner and the ranks meet in the
one SUM all-reduce of dist.py; the lexicographic reduce must give every
rank the single-process winner, including on cost ties."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_23838_b200.dist import best_row, pack, shard_range, unpack


def test_shard_range_partitions():
    for n in (0, 1, 7, 31, 1024, 1048864):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(got[i][1] == got[i + 1][0] for i in range(w - 1))
            assert max(e - b for b, e in got) - min(e - b for b, e in got) <= 1


def test_lexicographic_reduce_breaks_ties_like_reference():
    # equal cost, finish decides; equal (cost, finish): priority, then serial
    rows = np.stack([pack(50.0, 12.0, 2, 30), pack(50.0, 12.0, 0, 99), pack(50.0, 11.0, 2, 400),
                     np.zeros(4, dtype=np.uint64)])
    assert unpack(rows[best_row(rows)]) == (50.0, 11.0, 2, 400)
    rows[2] = pack(50.0, 12.0, 0, 98)
    assert unpack(rows[best_row(rows)]) == (50.0, 12.0, 0, 98)
    # an element-wise min would have mixed fields across rows
    assert best_row(np.zeros((3, 4), dtype=np.uint64)) == -1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, window, cap, q):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers import instance

    from oracle.oracle import Oracle
    from paper_2604_23838_b200.dist import WORDS, minloc_allreduce
    from paper_2604_23838_b200.state import State as HostState

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = instance(name)
    st = HostState(inst)
    o = Oracle(inst, nthreads=2)
    n = o.score(st, window, cap, serials=[])["n"]
    b, e = shard_range(n, rank, world)
    table = torch.zeros((world, WORDS), dtype=torch.int64)
    r = o.score(st, window, cap, serials=list(range(b, e)))
    if r["best"] is not None:
        table[rank] = torch.from_numpy(pack(*r["best"]).view(np.int64))
    rows = minloc_allreduce(table, rank)
    q.put((rank, unpack(rows[best_row(rows)])))
    dist.destroy_process_group()


@pytest.mark.parametrize("name,window,cap", [("trap", 3, None), ("trap", 1, None), ("async_small", 3, 3)])
def test_two_rank_decision_matches_single(name, window, cap):
    from helpers import instance

    from oracle.oracle import Oracle
    from paper_2604_23838_b200.state import State as HostState

    inst = instance(name)
    want = Oracle(inst, nthreads=2).score(HostState(inst), window, cap)["best"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, window, cap, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1] == tuple(want)
