"""paper_2604_23838_b200 — B200-native look-ahead candidate evaluator for the
PuzzRL multiplexing scheduler (arxiv 2604.23838, reference package `rlmux`).

Public surface (mirrors rlmux): lookahead_schedule, greedy_schedule,
serial_schedule, brute_force_schedule, simulate (+ simulate_batch),
Instance and the domain types; graphgen builds Sub-Stage Graphs from
rollout tables on the GPU; `Evaluator` is the C-ABI handle.
"""

from .model import (  # noqa: F401
    DEFAULT_LATENCY,
    FULL_ALLOCATION,
    Candidate,
    Exclusive,
    Instance,
    Merge,
    MemoryPressureError,
    Multiplex,
    OracleLimitError,
    PipelineSpec,
    ResourceAllocation,
    Schedule,
    SchedulingError,
    SlowdownModel,
    SlowdownTable,
    SubStage,
    SubStageGraph,
    SubStageKind,
    TimedAction,
    bucketize,
    complement_allocation,
    default_model,
    default_table,
    feasible,
    merged_estimate,
    migration_cost,
)
from .instance_io import as_instance, load_instance, load_instances, save_instance  # noqa: F401
from .scheduler import brute_force_schedule, drive, greedy_schedule, lookahead_schedule, serial_schedule  # noqa: F401
from .sim import SimulationReport, simulate, simulate_batch  # noqa: F401

__version__ = "0.1.0"
