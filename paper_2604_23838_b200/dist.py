"""Candidate sharding across GPUs and the one collective per decision.

Every rank holds the same decision state (SPMD replicas of the same
deterministic decision loop) and scores part `rank` of `world` of the
candidate set: every world-th block of 32 consecutive serials of each class
(multiplex, merges, exclusive), starting at block `rank` (`part_serials`,
the library's RLX_F_SHARD). Per class the blocks interleave, so every rank
gets the same mix of merge targets, pipelines and follow-up counts —
cost-balanced without a cost model (a merge costs 3(1+F) passes against 3
for the others, and F varies by target).

The shard winners are combined with ONE all-reduce: each rank writes its
packed 5-word row (cost bits, finish bits, priority<<61|serial, valid,
lowest failing serial<<8|code or ~0) into row `rank` of a zeroed
[world, 5] int64 buffer and a SUM all-reduce hands every rank all rows,
which it reduces lexicographically — identical on every rank, so all ranks
apply the same winner without a broadcast. (An element-wise MIN all-reduce
would mix fields of different ranks and break the reference's tie order,
SURVEY.md §8(e).) If any rank saw a failing candidate, every rank raises the
reference's exception for the globally lowest failing serial — the one the
reference's serial scan raises on. Over NCCL the buffer stays on the
device: the CUDA library writes the shard row straight into it
(RlxDecideArgs.dev_key_out).
"""

from __future__ import annotations

import numpy as np

WORDS = 5
BLOCK_SHIFT = 5  # = kShardBlockShift (csrc/rlx_abi.cu)
_MASK61 = (1 << 61) - 1
_NONE = (1 << 64) - 1


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [b, e) of n serials for `rank` (sizes differ by <= 1)."""
    q, r = divmod(n, world)
    b = rank * q + min(rank, r)
    return b, b + q + (1 if rank < r else 0)


def part_serials(counts, rank: int, world: int, shift: int = BLOCK_SHIFT) -> np.ndarray:
    """The serials part `rank` of `world` scores (RLX_F_SHARD): per class of
    `counts` = (n_multiplex, n_merge, n_exclusive), every world-th block of
    2**shift serials starting at block `rank`."""
    out = []
    s0 = 0
    for n in counts:
        s = np.arange(n, dtype=np.int64)
        out.append(s0 + s[(s >> shift) % world == rank])
        s0 += n
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


def first_error(rows: np.ndarray):
    """(serial, device code) of the lowest failing candidate over all rows of
    a [world, 5] uint64 table, or None."""
    e = rows[:, 4]
    e = e[e != np.uint64(_NONE)]
    if e.size == 0:
        return None
    m = int(e.min())
    return m >> 8, m & 0xFF


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


def pack(cost: float, finish: float, priority: int, serial: int, err: int | None = None) -> np.ndarray:
    """(cost, finish, priority, serial) -> the 5-word row: include/rlx.h
    RlxKey (costs are >= 0 doubles, so their bit patterns order as u64)
    plus the shard's lowest failing candidate (serial << 8 | code, or ~0)."""
    w = np.zeros(WORDS, dtype=np.uint64)
    w[0:2] = np.array([cost + 0.0, finish + 0.0], dtype=np.float64).view(np.uint64)
    w[2] = (int(priority) << 61) | int(serial)
    w[3] = 1
    w[4] = np.uint64(_NONE if err is None else err)
    return w


def empty_row(err: int | None = None) -> np.ndarray:
    """The row of a shard without candidates (or whose candidates all failed)."""
    w = np.zeros(WORDS, dtype=np.uint64)
    w[0:3] = np.uint64(_NONE)
    w[4] = np.uint64(_NONE if err is None else err)
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
        from .native import raise_device_error

        ev = self.ev
        self.table.zero_()
        self.torch.cuda.synchronize(self.table.device)
        row_ptr = self.table.data_ptr() + self.rank * WORDS * 8
        # one plan per decision; the library writes this rank's row (best key
        # and lowest failing serial) into the table even when its part fails,
        # so every rank reaches the all-reduce and raises the same error
        try:
            d = ev.decide(state, self.window, self.max_merge, part=(self.rank, self.world), dev_key_ptr=row_ptr)
            n = d.n_candidates
        except (RuntimeError, KeyError) as exc:
            if getattr(exc, "serial", None) is None:
                raise
            n = ev.last_n_candidates
        if n == 0:
            return None
        rows = minloc_allreduce(self.table, self.rank, self.group)
        fail = first_error(rows)
        if fail is not None:
            raise_device_error(fail[1], fail[0])
        i = best_row(rows)
        cost, fin, prio, serial = unpack(rows[i])
        action = ev.decode(serial)
        if self.log is not None:
            self.log.append({"now": state.now, "n": n, "key": [cost, fin, prio, serial], "action": action})
        return action
