"""Candidate sharding across GPUs and the one collective per decision.

Every rank holds the same decision state (SPMD replicas of the same
deterministic decision loop), scores a contiguous block of the global
serial range, and the shard winners are combined with ONE all-reduce: each
rank writes its packed 4-word key (cost bits, finish bits,
priority<<61|serial, valid) into row `rank` of a zeroed [world, 4] int64
buffer and a SUM all-reduce hands every rank all rows, which it reduces
lexicographically — identical on every rank, so all ranks apply the same
winner without a broadcast. (An element-wise MIN all-reduce would mix
fields of different ranks and break the reference's tie order,
SURVEY.md §8(e).) Over NCCL the buffer stays on the device: the CUDA
library writes the shard key straight into it (RlxDecideArgs.dev_key_out).
"""

from __future__ import annotations

import numpy as np

WORDS = 4
_MASK61 = (1 << 61) - 1


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [b, e) of n serials for `rank` (sizes differ by <= 1)."""
    q, r = divmod(n, world)
    b = rank * q + min(rank, r)
    return b, b + q + (1 if rank < r else 0)


def best_row(rows: np.ndarray) -> int:
    """Index of the lexicographically smallest valid row of a [world, 4]
    uint64 key table, or -1."""
    best = -1
    for i in range(rows.shape[0]):
        r = rows[i]
        if not r[3]:
            continue
        if best < 0 or tuple(int(x) for x in r[:3]) < tuple(int(x) for x in rows[best][:3]):
            best = i
    return best


def pack(cost: float, finish: float, priority: int, serial: int) -> np.ndarray:
    """(cost, finish, priority, serial) -> the 4-word key of include/rlx.h
    RlxKey (costs are >= 0 doubles, so their bit patterns order as u64)."""
    w = np.zeros(WORDS, dtype=np.uint64)
    w[0:2] = np.array([cost + 0.0, finish + 0.0], dtype=np.float64).view(np.uint64)
    w[2] = (int(priority) << 61) | int(serial)
    w[3] = 1
    return w


def unpack(row) -> tuple:
    """(cost, finish, priority, serial) of a packed key row."""
    w = np.asarray(row, dtype=np.uint64)
    cost = float(w[0:1].view(np.float64)[0])
    fin = float(w[1:2].view(np.float64)[0])
    ps = int(w[2])
    return cost, fin, ps >> 61, ps & _MASK61


def minloc_allreduce(table, rank: int, group=None):
    """SUM all-reduce of a [world, 4] int64 tensor where only row `rank` is
    set; returns the combined table as uint64 numpy."""
    import torch.distributed as dist

    dist.all_reduce(table, op=dist.ReduceOp.SUM, group=group)
    return table.cpu().numpy().view(np.uint64)


class ShardedChooser:
    """`drive` chooser for one rank of a multi-GPU decision."""

    def __init__(self, evaluator, window, max_merge, group, log=None):
        import torch
        import torch.distributed as dist

        self.ev = evaluator
        self.window = window
        self.max_merge = max_merge
        self.group = group
        self.log = log
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        dev = torch.device("cuda", evaluator.device)
        self.table = torch.zeros((self.world, WORDS), dtype=torch.int64, device=dev)
        self.torch = torch

    def __call__(self, state):
        ev = self.ev
        self.table.zero_()
        self.torch.cuda.synchronize(self.table.device)
        row_ptr = self.table.data_ptr() + self.rank * WORDS * 8
        # one plan per decision: the library sizes block `rank` of `world`
        # from the candidate count it enumerates (same as shard_range)
        d = ev.decide(state, self.window, self.max_merge, part=(self.rank, self.world), dev_key_ptr=row_ptr)
        n = d.n_candidates
        if n == 0:
            return None
        rows = minloc_allreduce(self.table, self.rank, self.group)
        i = best_row(rows)
        cost, fin, prio, serial = unpack(rows[i])
        action = ev.decode(serial)
        if self.log is not None:
            self.log.append({"now": state.now, "n": n, "key": [cost, fin, prio, serial], "action": action})
        return action
