"""Sub-Stage Graph construction from per-rollout length tables, on the GPU
(SURVEY.md §8(f)#2).

The reference turns a pipeline's sample batch into its Sub-Stage Graph in
pure Python: `expand_to_trace` replays every worker's cohort step by step
(rlmux/workload.py:275-392) and `construct_graph` segments each worker's
step records into bucket-stable rollout sub-stages and adds the Reference /
Training barrier (rlmux/graph.py:206-403). At config 5 that takes 77-114 s.
Here the replay and the segmentation run in `librlx.so` (csrc/rlx_graph.cu,
one warp per (pipeline, worker) cohort, one call for all pipelines); this
module only holds the tables and assembles SubStage rows from the
segments, in the reference's node order.

    batch = generate_synthetic(GeneratorConfig(batch=8192, workers=64, ...), seed=100)
    graph = construct_graph(batch)                     # one pipeline
    graphs = construct_graphs([b0, b1, ...])           # one device call
    inst = build_config(5)                             # BASELINE.json configs

`generate_synthetic` draws the same numbers as the reference generator
(workload.py:216-262; same numpy Generator, same draw order), so the
synthetic instances equal the reference's. Not reproduced: SubStage
`sample_ids` (the still-active sample sets of the enrichment replay) — they
are metadata that no scheduling path reads, and are left empty.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .model import (
    DEFAULT_BUCKET_BOUNDS,
    DEFAULT_LATENCY,
    DEFAULT_MEM_FRACTIONS,
    KIND_ORDER,
    Instance,
    PipelineSpec,
    SubStage,
    SubStageGraph,
    SubStageKind,
    default_model,
)

DEFAULT_TURN_PROBS = {1: 0.5, 2: 0.3, 3: 0.1, 4: 0.06, 5: 0.04}  # workload.py:176
DEFAULT_STABILITY_WINDOW = 10  # graph.py:27


@dataclass(frozen=True)
class GeneratorConfig:
    """Distribution knobs of a synthetic pipeline batch (workload.py:179-212)."""

    batch: int = 64
    workers: int = 1
    decode_median: float = 80.0
    decode_sigma: float = 1.0
    decode_max: int = 2000
    prompt_median: float = 128.0
    prompt_sigma: float = 0.3
    turn_probs: dict = field(default_factory=lambda: dict(DEFAULT_TURN_PROBS))
    turn_prefill_median: float = 200.0
    turn_prefill_sigma: float = 0.4
    tool_prob: float = 0.0
    tool_latency_mean: float = 0.0
    stages: tuple = ("rollout", "reference", "training")
    model_params: float = 4e9
    device_peak_flops: float = 1e15
    prefill_mfu: float = 0.4
    pipeline_id: str = "p0"

    def __post_init__(self) -> None:
        if self.decode_median <= 0 or self.prompt_median <= 0 or self.turn_prefill_median <= 0:
            raise ValueError("distribution medians must be positive")
        if min(self.decode_sigma, self.prompt_sigma, self.turn_prefill_sigma) < 0:
            raise ValueError("distribution sigmas must be non-negative")
        if self.tool_latency_mean < 0 or not 0 <= self.tool_prob <= 1:
            raise ValueError("invalid tool distribution parameters")
        if self.batch < 1 or self.workers < 1 or self.batch % self.workers != 0:
            raise ValueError("batch must be a positive multiple of workers")
        total = sum(self.turn_probs.values())
        if not self.turn_probs or abs(total - 1.0) > 1e-9 or min(self.turn_probs) < 1:
            raise ValueError("turn_probs must be a distribution over turn counts >= 1")


@dataclass
class RolloutBatch:
    """One pipeline's sample batch as flat tables (the reference's
    PipelineSpec, workload.py:75-110): per sample its prompt tokens and a
    CSR range of turns (prefill injected at the turn, decode tokens, tool
    latency after the turn)."""

    pipeline_id: str
    model_params: float
    dp_workers: int
    stages: tuple
    prompt: np.ndarray        # int64 [n]
    turn_off: np.ndarray      # int32 [n + 1]
    turn_prefill: np.ndarray  # int64 [turns]
    turn_decode: np.ndarray   # int64 [turns]
    turn_tool: np.ndarray     # float64 [turns]
    device_peak_flops: float = 1e15
    prefill_mfu: float = 0.4
    worker_of: np.ndarray | None = None  # int32 [n]; None: round robin (workload.py round_robin_assignment)

    @property
    def n_samples(self) -> int:
        return len(self.prompt)

    def spec(self) -> PipelineSpec:
        return PipelineSpec(self.pipeline_id, self.model_params, self.device_peak_flops, self.prefill_mfu)


def _lognormal_int(rng, median: float, sigma: float, lo: int, hi: int) -> int:
    value = median * math.exp(sigma * rng.standard_normal()) if sigma > 0 else median
    return int(min(max(round(value), lo), hi))


def generate_synthetic(config: GeneratorConfig, seed: int) -> RolloutBatch:
    """A synthetic batch, drawn exactly like the reference generator
    (workload.py:216-262): per sample the prompt, the turn count, then per
    turn its prefill (turns after the first), decode and tool latency."""
    rng = np.random.default_rng(seed)
    counts = sorted(config.turn_probs)
    p = np.array([config.turn_probs[k] for k in counts], dtype=float)
    p = p / p.sum()
    prompt = np.empty(config.batch, dtype=np.int64)
    off = [0]
    pre, dec, tool = [], [], []
    tool_on = config.tool_latency_mean > 0
    for sid in range(config.batch):
        prompt[sid] = _lognormal_int(rng, config.prompt_median, config.prompt_sigma, 1, 1 << 20)
        n_turns = int(rng.choice(counts, p=p))
        for t in range(n_turns):
            pre.append(_lognormal_int(rng, config.turn_prefill_median, config.turn_prefill_sigma, 1, 1 << 20)
                       if t > 0 else 0)
            dec.append(_lognormal_int(rng, config.decode_median, config.decode_sigma, 1, config.decode_max))
            tl = 0.0
            if t < n_turns - 1 and tool_on and rng.random() < config.tool_prob:
                tl = float(rng.exponential(config.tool_latency_mean))
            tool.append(tl)
        off.append(len(dec))
    return RolloutBatch(pipeline_id=config.pipeline_id, model_params=config.model_params, dp_workers=config.workers,
                        stages=tuple(config.stages), prompt=prompt, turn_off=np.array(off, dtype=np.int32),
                        turn_prefill=np.array(pre, dtype=np.int64), turn_decode=np.array(dec, dtype=np.int64),
                        turn_tool=np.array(tool, dtype=np.float64), device_peak_flops=config.device_peak_flops,
                        prefill_mfu=config.prefill_mfu)


def batch_from_spec(spec, assignment: dict | None = None) -> RolloutBatch:
    """The tables of a reference `rlmux` PipelineSpec (drop-in input)."""
    samples = sorted(spec.samples, key=lambda s: s.sample_id)
    off, pre, dec, tool = [0], [], [], []
    for s in samples:
        for t in s.turns:
            pre.append(t.prefill_tokens)
            dec.append(t.decode_tokens)
            tool.append(float(t.tool_latency))
        off.append(len(dec))
    worker_of = None
    if assignment is not None:
        worker_of = np.array([assignment[s.sample_id] for s in samples], dtype=np.int32)
    elif [s.sample_id for s in samples] != list(range(len(samples))):
        worker_of = np.array([s.sample_id % spec.dp_workers for s in samples], dtype=np.int32)
    return RolloutBatch(pipeline_id=spec.pipeline_id, model_params=spec.model_params, dp_workers=spec.dp_workers,
                        stages=tuple(spec.stages), prompt=np.array([s.prompt_tokens for s in samples], dtype=np.int64),
                        turn_off=np.array(off, dtype=np.int32), turn_prefill=np.array(pre, dtype=np.int64),
                        turn_decode=np.array(dec, dtype=np.int64), turn_tool=np.array(tool, dtype=np.float64),
                        device_peak_flops=spec.device_peak_flops, prefill_mfu=spec.prefill_mfu, worker_of=worker_of)


@dataclass
class BuildStats:
    kernel_ms: float = 0.0   # replay + segmentation kernels (CUDA events)
    records: int = 0         # forward-step records replayed
    segments: int = 0        # rollout sub-stages


def construct_graphs(batches, latency_models=None, stability_window: int = DEFAULT_STABILITY_WINDOW,
                     bucket_bounds=DEFAULT_BUCKET_BOUNDS, mem_fractions: dict | None = None, device: int = 0,
                     stats: BuildStats | None = None) -> list:
    """One SubStageGraph per batch (construct_graph(expand_to_trace(spec),
    spec=spec), graph.py:285-403), all pipelines replayed and segmented in
    one device call."""
    from .native import _raise, load_library

    if stability_window < 1:
        raise ValueError("stability_window must be >= 1")
    bounds = tuple(int(b) for b in bucket_bounds)
    if not bounds or bounds[0] != 0 or list(bounds) != sorted(set(bounds)):
        raise ValueError(f"bucket bounds must be strictly increasing from 0, got {bounds}")
    lats = [dict(DEFAULT_LATENCY) if latency_models is None or latency_models[i] is None else dict(latency_models[i])
            for i in range(len(batches))]
    lib = load_library()
    keep = []
    tabs = (abi.RlxRolloutTables * len(batches))()
    for i, b in enumerate(batches):
        lat = lats[i]
        for k in (0, 1, 2):
            if k not in lat:
                raise KeyError(k)
        arrs = [np.ascontiguousarray(b.prompt, dtype=np.int64), np.ascontiguousarray(b.turn_off, dtype=np.int32),
                np.ascontiguousarray(b.turn_prefill, dtype=np.int64), np.ascontiguousarray(b.turn_decode, dtype=np.int64),
                np.ascontiguousarray(b.turn_tool, dtype=np.float64)]
        wo = None if b.worker_of is None else np.ascontiguousarray(b.worker_of, dtype=np.int32)
        keep += arrs + [wo]
        t = tabs[i]
        t.n_samples = b.n_samples
        t.n_workers = b.dp_workers
        t.worker_of = None if wo is None else wo.ctypes.data_as(C.POINTER(C.c_int32))
        t.prompt = arrs[0].ctypes.data_as(C.POINTER(C.c_int64))
        t.turn_off = arrs[1].ctypes.data_as(C.POINTER(C.c_int32))
        t.turn_prefill = arrs[2].ctypes.data_as(C.POINTER(C.c_int64))
        t.turn_decode = arrs[3].ctypes.data_as(C.POINTER(C.c_int64))
        t.turn_tool = arrs[4].ctypes.data_as(C.POINTER(C.c_double))
        for k in range(5):
            t.latency[k] = float(lat.get(k, float("nan")))
    bnd = (C.c_int32 * len(bounds))(*bounds)
    res = C.c_void_p()
    rc = lib.rlx_graph_build(int(device), len(batches), tabs, bnd, len(bounds), int(stability_window), C.byref(res))
    try:
        if rc != 0:
            _raise(rc, (lib.rlx_graph_error(res) or b"").decode())
        graphs = []
        km = C.c_double()
        nrec = C.c_int64()
        lib.rlx_graph_stats(res, C.byref(km), C.byref(nrec))
        nseg_total = 0
        for i, b in enumerate(batches):
            n = C.c_int64()
            lib.rlx_graph_segments(res, i, None, 0, C.byref(n))
            segs = (abi.RlxSegment * max(n.value, 1))()
            lib.rlx_graph_segments(res, i, segs, n.value, C.byref(n))
            nseg_total += n.value
            graphs.append(_assemble(b, segs[: n.value], lats[i], mem_fractions))
        if stats is not None:
            stats.kernel_ms, stats.records, stats.segments = km.value, nrec.value, nseg_total
        return graphs
    finally:
        lib.rlx_graph_free(res)


def construct_graph(batch, latency_model=None, **kw) -> SubStageGraph:
    return construct_graphs([batch], None if latency_model is None else [latency_model], **kw)[0]


def _assemble(b: RolloutBatch, segs, latency: dict, mem_fractions) -> SubStageGraph:
    """SubStage rows in the reference's order: rollout sub-stages worker by
    worker (chained), then one Reference per worker after its last rollout
    sub-stage, then one Training per worker behind every worker's tail
    (the gradient-sync barrier, graph.py:363-395)."""
    mem = dict(DEFAULT_MEM_FRACTIONS)
    if mem_fractions:
        mem.update(mem_fractions)
    pid = b.pipeline_id
    nodes, edges, last = {}, set(), {}
    prev, prev_w = None, None
    for s in segs:
        if s.worker != prev_w:
            prev, prev_w = None, s.worker
        kind = KIND_ORDER[s.kind]
        sid = f"{pid}/w{s.worker}/r{s.seq:03d}"
        nodes[sid] = SubStage(id=sid, pipeline_id=pid, worker_id=int(s.worker), kind=kind, duration=s.duration,
                              mem_fraction=mem[kind], step_span=(int(s.step_lo), int(s.step_hi)),
                              remaining_decode_tokens=int(s.decode), active_requests=int(s.active0),
                              context_tokens=int(s.context0), token_total=int(s.tokens))
        if prev is not None:
            edges.add((prev, sid))
        prev = sid
        last[int(s.worker)] = sid
    tail = dict(last)
    if "reference" in b.stages:
        if 3 not in latency:
            raise ValueError("latency model has no entry for the reference stage")
        for w, t in sorted(tail.items()):
            sid = f"{pid}/w{w}/ref"
            nodes[sid] = SubStage(id=sid, pipeline_id=pid, worker_id=w, kind=SubStageKind.REFERENCE,
                                  duration=latency[3], mem_fraction=mem[SubStageKind.REFERENCE])
            edges.add((t, sid))
        tail = {w: f"{pid}/w{w}/ref" for w in tail}
    if "training" in b.stages:
        if 4 not in latency:
            raise ValueError("latency model has no entry for the training stage")
        for w in sorted(tail):
            sid = f"{pid}/w{w}/train"
            nodes[sid] = SubStage(id=sid, pipeline_id=pid, worker_id=w, kind=SubStageKind.TRAINING,
                                  duration=latency[4], mem_fraction=mem[SubStageKind.TRAINING])
            for t in tail.values():
                edges.add((t, sid))
    return SubStageGraph(pipeline_id=pid, nodes=nodes, edges=edges, spec=b.spec(), latency_model=dict(latency))


# ---------------------------------------------------------------------------
# The BASELINE.json config instances (SURVEY.md §8(d) recipes)


def asyncify(g: SubStageGraph) -> SubStageGraph:
    """Config-3 'async' recipe (builder-defined): drop the
    cross-worker Training barrier edges (graph.py:393-395), keeping the
    same-worker ref -> train edge, and add an independent mid-step Training
    node per worker, ready at t=0 (rlmux/fixtures.py:131-138 pattern)."""
    nodes = dict(g.nodes)
    edges = {(a, b) for a, b in g.edges
             if not (nodes[b].kind is SubStageKind.TRAINING and nodes[a].worker_id != nodes[b].worker_id)}
    for w in sorted({n.worker_id for n in g.nodes.values()}):
        sid = f"{g.pipeline_id}/w{w}/mid"
        nodes[sid] = SubStage(id=sid, pipeline_id=g.pipeline_id, worker_id=w, kind=SubStageKind.TRAINING,
                              duration=g.latency_model[4], mem_fraction=0.6)
    return SubStageGraph(pipeline_id=g.pipeline_id, nodes=nodes, edges=edges, spec=g.spec,
                         latency_model=dict(g.latency_model))


def config_batches(k: int) -> list:
    """The sample batches of BASELINE.json configs[k-1] (seeds and shapes
    of SURVEY.md §8(d))."""
    def pipe(pid, params, seed, batch, workers, sigma=1.0, **kw):
        return generate_synthetic(GeneratorConfig(batch=batch, workers=workers, model_params=params, decode_sigma=sigma,
                                                  pipeline_id=pid, **kw), seed)

    if k == 1:
        return [pipe("qwen8b", 8e9, 0, 256, 8)]
    if k == 2:
        return [pipe("qwen8b", 8e9, 1, 512, 16), pipe("qwen14b", 14e9, 2, 512, 16)]
    if k == 3:
        return [pipe(f"p{i}", p, 10 + i, 1024, 32, sigma=1.5) for i, p in enumerate((4e9, 8e9, 14e9, 32e9))]
    if k == 4:
        return [pipe(f"a{i}", p, 30 + i, 4096, 64, sigma=1.0, tool_prob=0.5, tool_latency_mean=2.0)
                for i, p in enumerate((0.6e9, 4e9, 8e9, 14e9))]
    if k == 5:
        return [pipe(f"p{i}", p, 100 + i, 8192, 64, sigma=1.5)
                for i, p in enumerate((4e9, 8e9, 8e9, 14e9, 14e9, 32e9, 4e9, 8e9))]
    raise ValueError(k)


def build_config(k: int, device: int = 0, batches=None, stats: BuildStats | None = None) -> Instance:
    """The config-k instance built on the GPU (tests/golden/instances holds
    the reference generator's output for comparison)."""
    graphs = construct_graphs(batches if batches is not None else config_batches(k), device=device, stats=stats)
    if k == 3:
        graphs = [asyncify(g) for g in graphs]
    return Instance(graphs=graphs, model=default_model())
