"""Multi-rank decision on CPU (gloo, world_size 2): each rank scores its
part of the serials (dist.part_serials — the library's block-cyclic
RLX_F_SHARD), packs its shard winner and the ranks meet in the one SUM
all-reduce of dist.py; the lexicographic reduce must give every rank the
single-process winner, including on cost ties, and a failing candidate on
one rank must make every rank raise for the globally lowest failing serial."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_23838_b200.dist import best_row, empty_row, first_error, pack, part_serials, shard_range, unpack


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
                     empty_row()])
    assert unpack(rows[best_row(rows)]) == (50.0, 11.0, 2, 400)
    rows[2] = pack(50.0, 12.0, 0, 98)
    assert unpack(rows[best_row(rows)]) == (50.0, 12.0, 0, 98)
    # an element-wise min would have mixed fields across rows
    assert best_row(np.zeros((3, 5), dtype=np.uint64)) == -1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, window, cap, q, fail=False):
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
    counts = o.counts(st, window, cap)
    mine = part_serials(counts, rank, world)
    table = torch.zeros((world, WORDS), dtype=torch.int64)
    r = o.score(st, window, cap, serials=mine.tolist())
    # rank 1 reports a (synthetic) failing candidate: both ranks must see it
    err = (5 << 8 | 1) if rank == 1 and fail else None
    row = pack(*r["best"], err=err) if r["best"] is not None else empty_row(err)
    table[rank] = torch.from_numpy(row.view(np.int64))
    rows = minloc_allreduce(table, rank)
    q.put((rank, unpack(rows[best_row(rows)]), first_error(rows)))
    dist.destroy_process_group()


def test_part_serials_cover_each_class_once():
    for counts in ((288, 1048544, 32), (32046, 32256, 512), (0, 5, 0), (7, 0, 3), (31, 33, 65)):
        for w in (1, 2, 3, 8):
            parts = [part_serials(counts, r, w) for r in range(w)]
            allp = np.sort(np.concatenate(parts))
            assert (allp == np.arange(sum(counts))).all()
            # every class splits into near-equal parts (block granularity)
            for lo, n in ((0, counts[0]), (counts[0], counts[1]), (counts[0] + counts[1], counts[2])):
                sizes = [int(((p >= lo) & (p < lo + n)).sum()) for p in parts]
                assert max(sizes) - min(sizes) <= 32


def test_first_error_is_the_lowest_failing_serial():
    rows = np.stack([pack(5.0, 1.0, 0, 3), empty_row(900 << 8 | 1), pack(4.0, 1.0, 1, 700, err=750 << 8 | 16)])
    assert first_error(rows) == (750, 16)
    assert first_error(np.stack([pack(5.0, 1.0, 0, 3), empty_row()])) is None


def _run_ranks(name, window, cap, fail=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, window, cap, q, fail)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, best, err = q.get(timeout=300)
        got[rank] = (best, err)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("name,window,cap", [("trap", 3, None), ("trap", 1, None), ("async_small", 3, 3)])
def test_two_rank_decision_matches_single(name, window, cap):
    from helpers import instance

    from oracle.oracle import Oracle
    from paper_2604_23838_b200.state import State as HostState

    inst = instance(name)
    want = Oracle(inst, nthreads=2).score(HostState(inst), window, cap)["best"]
    got = _run_ranks(name, window, cap)
    assert got[0][0] == got[1][0] == tuple(want)
    assert got[0][1] is got[1][1] is None


def test_two_rank_error_reaches_every_rank():
    got = _run_ranks("trap", 3, None, fail=True)
    assert got[0][1] == got[1][1] is not None
    assert got[0][1][1] == 1
