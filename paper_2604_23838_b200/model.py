"""Host-side mirror of the reference's domain types and cost model.

Everything here is the *interface* a user of the reference `rlmux` package
already programs against (same names, fields, argument meaning and error
classes), re-stated for this framework so it runs without the reference:

* sub-stage kinds / constants / `SubStage` / `SubStageGraph`
  (rlmux/graph.py:26-191)
* `ResourceAllocation`, grids, `feasible`, `complement_allocation`, the
  bilinear `SlowdownModel` and the default table (rlmux/slowdown.py:18-272)
* actions, `TimedAction`, `Schedule`, `Instance`, errors
  (rlmux/scheduler.py:43-151)
* `merged_estimate` / `migration_cost` (rlmux/scheduler.py:174-199)

The arithmetic that feeds the device path (bilinear interpolation,
complement, merged duration, migration cost) is written to evaluate in
exactly the reference's IEEE-754 binary64 operation order, because the
chooser's tie-breaks depend on bit-identical costs.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

EPS = 1e-9  # rlmux/scheduler.py:43
MUX_SM_GRID = (0.25, 0.50, 0.75)  # rlmux/scheduler.py:46
SM_GRID = (0.25, 0.50, 0.75, 1.00)  # rlmux/slowdown.py:18
MEM_GRID = (0.20, 0.40, 0.60, 0.80)  # rlmux/slowdown.py:19
DEFAULT_HEADROOM = 0.05  # rlmux/slowdown.py:20
DEFAULT_BUCKET_BOUNDS = (0, 128, 1024)  # rlmux/graph.py:26
REFERENCE_INDEX = 3  # rlmux/workload.py:23
TRAINING_INDEX = 4  # rlmux/workload.py:24
DEFAULT_LATENCY = {0: 0.02, 1: 0.05, 2: 0.18, REFERENCE_INDEX: 4.0, TRAINING_INDEX: 10.0}  # workload.py:28


class SchedulingError(RuntimeError):
    """An action cannot be applied, the driver stalled, or a window estimate
    did not converge (rlmux/scheduler.py:51)."""


class MemoryPressureError(SchedulingError):
    """rlmux/scheduler.py:55"""


class OracleLimitError(RuntimeError):
    """rlmux/scheduler.py:59"""


class TableValidationError(ValueError):
    """rlmux/slowdown.py:34"""


def bucketize(tokens: int, bounds: tuple[int, ...] = DEFAULT_BUCKET_BOUNDS) -> int:
    """Token count -> half-open bucket index, last bucket unbounded
    (rlmux/graph.py:59-66)."""
    if tokens < 0:
        raise ValueError(f"token count must be >= 0, got {tokens}")
    idx = 0
    for i, lo in enumerate(bounds):
        if tokens >= lo:
            idx = i
    return idx


class SubStageKind(enum.Enum):
    """rlmux/graph.py:69-76 (same values, same declaration order)."""

    PREFILL_BURST = "PrefillBurst"
    DECODE_LARGE = "DecodeLarge"
    DECODE_MEDIUM = "DecodeMedium"
    DECODE_SMALL = "DecodeSmall"
    REFERENCE = "Reference"
    TRAINING = "Training"
    TOOL_WAIT = "ToolWait"


KIND_ORDER = tuple(SubStageKind)  # device kind code = index in this tuple
KIND_CODE = {k: i for i, k in enumerate(KIND_ORDER)}

ROLLOUT_KINDS = frozenset(
    {SubStageKind.PREFILL_BURST, SubStageKind.DECODE_LARGE, SubStageKind.DECODE_MEDIUM, SubStageKind.DECODE_SMALL}
)
MERGEABLE_KINDS = frozenset({SubStageKind.DECODE_SMALL, SubStageKind.DECODE_MEDIUM})
DECODE_KIND_BY_BUCKET = {0: SubStageKind.DECODE_SMALL, 1: SubStageKind.DECODE_MEDIUM, 2: SubStageKind.DECODE_LARGE}
DEFAULT_MEM_FRACTIONS = {
    SubStageKind.PREFILL_BURST: 0.5,
    SubStageKind.DECODE_LARGE: 0.55,
    SubStageKind.DECODE_MEDIUM: 0.4,
    SubStageKind.DECODE_SMALL: 0.3,
    SubStageKind.REFERENCE: 0.5,
    SubStageKind.TRAINING: 0.6,
    SubStageKind.TOOL_WAIT: 0.05,
}


@dataclass(frozen=True)
class SubStage:
    """rlmux/graph.py:109-137."""

    id: str
    pipeline_id: str
    worker_id: int
    kind: SubStageKind
    duration: float
    mem_fraction: float
    step_span: tuple[int, int] = (0, 0)
    sample_ids: frozenset = frozenset()
    remaining_decode_tokens: int = 0
    active_requests: int = 0
    context_tokens: int = 0
    token_total: int = 0

    def __post_init__(self) -> None:
        if self.kind is SubStageKind.TOOL_WAIT:
            if self.duration < 0:
                raise ValueError(f"{self.id}: tool wait duration must be >= 0")
        elif self.duration <= 0:
            raise ValueError(f"{self.id}: duration must be positive")
        if not 0 < self.mem_fraction <= 1:
            raise ValueError(f"{self.id}: mem_fraction must be in (0, 1]")

    @property
    def is_rollout(self) -> bool:
        return self.kind in ROLLOUT_KINDS


@dataclass(frozen=True)
class PipelineSpec:
    """The fields of rlmux/workload.py:75-110 that the scheduling path reads
    (migration cost, scheduler.py:174-182)."""

    pipeline_id: str
    model_params: float
    device_peak_flops: float = 1e15
    prefill_mfu: float = 0.4


@dataclass
class SubStageGraph:
    """rlmux/graph.py:140-191 (edges as a set of (src, dst) id pairs)."""

    pipeline_id: str
    nodes: dict
    edges: set
    spec: PipelineSpec | None = None
    latency_model: dict = field(default_factory=dict)

    def __post_init__(self) -> None:
        for src, dst in self.edges:
            if src not in self.nodes or dst not in self.nodes:
                raise ValueError(f"edge ({src}, {dst}) references unknown node")

    def worker_ids(self) -> list[int]:
        return sorted({n.worker_id for n in self.nodes.values()})

    @property
    def total_tokens(self) -> int:
        return sum(n.token_total for n in self.nodes.values())


@dataclass(frozen=True)
class ResourceAllocation:
    """rlmux/slowdown.py:38-49."""

    sm_share: float
    mem_share: float

    def __post_init__(self) -> None:
        if not 0 < self.sm_share <= 1:
            raise ValueError(f"sm_share must be in (0, 1], got {self.sm_share}")
        if not 0 < self.mem_share <= 1:
            raise ValueError(f"mem_share must be in (0, 1], got {self.mem_share}")


FULL_ALLOCATION = ResourceAllocation(1.0, MEM_GRID[-1])  # rlmux/slowdown.py:52


def feasible(mem_a: float, mem_b: float, headroom: float = DEFAULT_HEADROOM) -> bool:
    """rlmux/slowdown.py:162-166."""
    if not 0 < mem_a <= 1 or not 0 < mem_b <= 1:
        raise ValueError("memory fractions must be in (0, 1]")
    return mem_a + mem_b <= 1.0 - headroom + 1e-12


def complement_allocation(alloc: ResourceAllocation, headroom: float = DEFAULT_HEADROOM) -> ResourceAllocation:
    """rlmux/slowdown.py:169-175."""
    sm = max(SM_GRID[0], min(1.0 - alloc.sm_share, 1.0))
    mem = max(0.05, 1.0 - alloc.mem_share - headroom)
    return ResourceAllocation(sm, mem)


def _bracket(grid, x):
    """Bracketing grid points + weight, clamped (rlmux/slowdown.py:109-120)."""
    if x <= grid[0]:
        return grid[0], grid[0], 0.0
    if x >= grid[-1]:
        return grid[-1], grid[-1], 0.0
    for lo, hi in zip(grid, grid[1:]):
        if lo <= x <= hi:
            return (lo, hi, 0.0) if lo == hi else (lo, hi, (x - lo) / (hi - lo))
    return grid[-1], grid[-1], 0.0


@dataclass
class SlowdownTable:
    """Factor grid keyed (kind, partner|None, alpha, mem) (rlmux/slowdown.py:57-106)."""

    entries: dict

    def validate(self) -> None:
        pairs = {(k, p) for k, p, _, _ in self.entries}
        for kind, partner in pairs:
            for a in SM_GRID:
                for m in MEM_GRID:
                    if (kind, partner, a, m) not in self.entries:
                        raise TableValidationError(f"missing grid point {kind.value} at alpha={a} mem={m}")
                    if self.entries[(kind, partner, a, m)] < 1.0:
                        raise TableValidationError(f"factor < 1.0 at {kind.value} alpha={a} mem={m}")


@dataclass
class SlowdownModel:
    """Bilinear view over a table (rlmux/slowdown.py:123-159)."""

    table: SlowdownTable

    def slowdown(self, kind_a: SubStageKind, kind_b: SubStageKind | None, alloc: ResourceAllocation) -> float:
        if kind_a is SubStageKind.TOOL_WAIT:
            return 1.0
        a_lo, a_hi, wa = _bracket(SM_GRID, alloc.sm_share)
        m_lo, m_hi, wm = _bracket(MEM_GRID, alloc.mem_share)
        e = self.table.entries
        try:
            f00 = e[(kind_a, kind_b, a_lo, m_lo)]
            f10 = e[(kind_a, kind_b, a_hi, m_lo)]
            f01 = e[(kind_a, kind_b, a_lo, m_hi)]
            f11 = e[(kind_a, kind_b, a_hi, m_hi)]
        except KeyError:
            partner = kind_b.value if kind_b else "-"
            raise KeyError(f"slowdown table has no rows for pair {kind_a.value}/{partner}") from None
        lo = f00 + (f10 - f00) * wa
        hi = f01 + (f11 - f01) * wa
        return lo + (hi - lo) * wm

    def max_factor(self) -> float:
        return max(self.table.entries.values())


# Default table fixture: same anchored curves as rlmux/slowdown.py:198-268.
_SM_CURVE = {
    SubStageKind.TRAINING: (2.70, 1.825, 1.30, 1.0),
    SubStageKind.REFERENCE: (2.30, 1.60, 1.22, 1.0),
    SubStageKind.PREFILL_BURST: (2.60, 1.75, 1.28, 1.0),
    SubStageKind.DECODE_LARGE: (2.40, 1.70, 1.25, 1.0),
    SubStageKind.DECODE_MEDIUM: (1.50, 1.25, 1.10, 1.0),
    SubStageKind.DECODE_SMALL: (1.08, 1.05, 1.02, 1.0),
    SubStageKind.TOOL_WAIT: (1.0, 1.0, 1.0, 1.0),
}
_MEM_CURVE = {
    SubStageKind.TRAINING: (1.45, 1.20, 1.08, 1.0),
    SubStageKind.REFERENCE: (1.35, 1.18, 1.07, 1.0),
    SubStageKind.PREFILL_BURST: (1.30, 1.15, 1.05, 1.0),
    SubStageKind.DECODE_LARGE: (1.70, 1.43, 1.18, 1.0),
    SubStageKind.DECODE_MEDIUM: (1.40, 1.20, 1.08, 1.0),
    SubStageKind.DECODE_SMALL: (1.15, 1.08, 1.03, 1.0),
    SubStageKind.TOOL_WAIT: (1.0, 1.0, 1.0, 1.0),
}
_COMPUTE_BOUND = frozenset(
    {SubStageKind.TRAINING, SubStageKind.REFERENCE, SubStageKind.PREFILL_BURST, SubStageKind.DECODE_LARGE}
)


def _cross(kind_a: SubStageKind, kind_b: SubStageKind | None) -> float:
    if kind_b is None or SubStageKind.TOOL_WAIT in (kind_a, kind_b):
        return 1.0
    ca, cb = kind_a in _COMPUTE_BOUND, kind_b in _COMPUTE_BOUND
    if ca and cb:
        return 1.0
    if cb:
        return 1.06
    if ca:
        return 1.03
    small = SubStageKind.DECODE_SMALL
    if kind_a is small and kind_b is small:
        return 1.12
    return 1.30 if small in (kind_a, kind_b) else 1.50


def default_table() -> SlowdownTable:
    entries = {}
    for kind in KIND_ORDER:
        for partner in (None, *KIND_ORDER):
            cross = _cross(kind, partner)
            for ai, alpha in enumerate(SM_GRID):
                for mi, memv in enumerate(MEM_GRID):
                    if kind is SubStageKind.TOOL_WAIT:
                        f = 1.0
                    elif partner is None and ai == 3 and mi == 3:
                        f = 1.0
                    else:
                        f = _SM_CURVE[kind][ai] * _MEM_CURVE[kind][mi] * cross
                    entries[(kind, partner, alpha, memv)] = f
    return SlowdownTable(entries)


def default_model() -> SlowdownModel:
    return SlowdownModel(default_table())


# ---------------------------------------------------------------------------
# Actions / schedules / instance (rlmux/scheduler.py:67-151)


@dataclass(frozen=True)
class Exclusive:
    node_id: str
    alloc: ResourceAllocation = FULL_ALLOCATION

    def members(self) -> tuple:
        return (self.node_id,)


@dataclass(frozen=True)
class Multiplex:
    node_a: str
    node_b: str
    alloc_a: ResourceAllocation

    def members(self) -> tuple:
        return (self.node_a, self.node_b)


@dataclass(frozen=True)
class Merge:
    member_ids: tuple
    target_worker: int

    def members(self) -> tuple:
        return self.member_ids


@dataclass(frozen=True)
class TimedAction:
    start: float
    action: object


@dataclass
class Schedule:
    actions: list
    policy: str = ""
    metadata: dict = field(default_factory=dict)


@dataclass(frozen=True)
class Candidate:
    """rlmux/scheduler.py:641-645; priority 0 multiplex, 1 merge, 2 exclusive."""

    serial: int
    priority: int
    action: object


@dataclass
class Instance:
    graphs: list
    model: SlowdownModel
    headroom: float = DEFAULT_HEADROOM
    realloc_penalty: float = 0.0
    default_migration_cost: float = 0.0
    merge_enabled: bool = True

    def __post_init__(self) -> None:
        ids = [g.pipeline_id for g in self.graphs]
        if len(set(ids)) != len(ids):
            raise ValueError(f"duplicate pipeline ids: {ids}")
        seen: set = set()
        for g in self.graphs:
            dup = seen & set(g.nodes)
            if dup:
                raise ValueError(f"node ids shared between pipelines: {sorted(dup)[:3]}")
            seen |= set(g.nodes)

    def workers(self) -> list[int]:
        out: set = set()
        for g in self.graphs:
            out.update(g.worker_ids())
        return sorted(out)

    def latency_model_for(self, pipeline_id: str) -> dict:
        for g in self.graphs:
            if g.pipeline_id == pipeline_id:
                return g.latency_model
        raise KeyError(pipeline_id)

    def spec_for(self, pipeline_id: str):
        for g in self.graphs:
            if g.pipeline_id == pipeline_id:
                return g.spec
        return None


def migration_cost(sub_stage: SubStage, spec) -> float:
    """KV recompute seconds: 2*params*context FLOPs at prefill MFU
    (rlmux/scheduler.py:174-182)."""
    if spec.prefill_mfu <= 0:
        raise ValueError("prefill_mfu must be positive")
    flops = 2.0 * spec.model_params * sub_stage.context_tokens
    return flops / (spec.prefill_mfu * spec.device_peak_flops)


def merged_estimate(members: list, latency_model: dict):
    """Perfect-dynamic-batching kind/duration of a merged fragment
    (rlmux/scheduler.py:185-199)."""
    tokens = sum(m.remaining_decode_tokens for m in members)
    active = sum(m.active_requests for m in members)
    if active <= 0:
        return members[0].kind, max(m.duration for m in members)
    bucket = bucketize(active)
    kind = DECODE_KIND_BY_BUCKET.get(bucket, SubStageKind.DECODE_LARGE)
    return kind, tokens * latency_model[bucket] / active
