"""Instance / state -> the flat arrays of the C-ABI (include/rlx.h).

`InstanceEncoding` is built once per instance: pipeline table, knobs and
the slowdown LUT. The LUT holds every factor the chooser can query —
FULL_ALLOCATION, the 12 Multiplex allocations (MUX_SM_GRID x MEM_GRID,
rlmux/scheduler.py:671-675) and their complements (slowdown.py:169-175) —
for all (kind, partner) pairs, evaluated here with the reference's own
bilinear op order so the device only does table lookups.

`GraphEncoding` is the static sub-stage graph the native execution state
(`state.State`, csrc/rlx_state.cpp) is created from; the per-decision
state the device consumes is a view of that native state, not a Python
re-encode.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from .model import (
    FULL_ALLOCATION,
    KIND_CODE,
    KIND_ORDER,
    MEM_GRID,
    MUX_SM_GRID,
    ResourceAllocation,
    complement_allocation,
)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def allocation_table(headroom: float) -> list:
    """Allocation index -> ResourceAllocation (include/rlx.h RLX_NALLOC layout)."""
    allocs = [FULL_ALLOCATION]
    mux = [ResourceAllocation(a, m) for a in MUX_SM_GRID for m in MEM_GRID]
    allocs += mux
    allocs += [complement_allocation(x, headroom) for x in mux]
    assert len(allocs) == abi.RLX_NALLOC
    return allocs


def build_lut(model, headroom: float) -> np.ndarray:
    allocs = allocation_table(headroom)
    lut = np.full((abi.RLX_NKIND, abi.RLX_NPARTNER, abi.RLX_NALLOC), np.nan, dtype=np.float64)
    partners = (None, *KIND_ORDER)
    for ki, kind in enumerate(KIND_ORDER):
        for pi, partner in enumerate(partners):
            for ai, alloc in enumerate(allocs):
                try:
                    lut[ki, pi, ai] = model.slowdown(kind, partner, alloc)
                except KeyError:
                    pass
    return lut


class InstanceEncoding:
    def __init__(self, instance):
        self.instance = instance
        graphs = instance.graphs
        self.pipe_ids = [g.pipeline_id for g in graphs]
        self.pipe_index = {p: i for i, p in enumerate(self.pipe_ids)}
        self.workers = instance.workers()
        self.worker_index = {w: i for i, w in enumerate(self.workers)}
        P = len(graphs)
        names = b""
        offs = []
        for p in self.pipe_ids:
            offs.append(len(names))
            names += p.encode("utf-8") + b"\0"
        self._names = names
        self.pipe_name_off = np.array(offs, dtype=np.int32)
        self.latency = np.zeros(P * 3, dtype=np.float64)
        self.latency_ok = np.zeros(P * 3, dtype=np.uint8)
        self.has_spec = np.zeros(P, dtype=np.uint8)
        self.params = np.zeros(P, dtype=np.float64)
        self.peak = np.ones(P, dtype=np.float64)
        self.mfu = np.ones(P, dtype=np.float64)
        for i, g in enumerate(graphs):
            for b in range(3):
                if b in g.latency_model:
                    self.latency[i * 3 + b] = float(g.latency_model[b])
                    self.latency_ok[i * 3 + b] = 1
            if g.spec is not None:
                if g.spec.prefill_mfu <= 0:
                    raise ValueError("prefill_mfu must be positive")
                self.has_spec[i] = 1
                self.params[i] = g.spec.model_params
                self.peak[i] = g.spec.device_peak_flops
                self.mfu[i] = g.spec.prefill_mfu
        self.worker_ids = np.array(self.workers, dtype=np.int32)
        self.lut = np.ascontiguousarray(build_lut(instance.model, instance.headroom).reshape(-1))
        allocs = allocation_table(instance.headroom)
        self.alloc_sm = np.array([a.sm_share for a in allocs], dtype=np.float64)
        self.alloc_mem = np.array([a.mem_share for a in allocs], dtype=np.float64)
        self.alloc_index = {}
        for i, a in enumerate(allocs[:13]):
            self.alloc_index.setdefault((a.sm_share, a.mem_share), i)
        self.allocs = allocs
        d = abi.RlxInstanceDesc()
        d.abi_version = abi.RLX_ABI_VERSION
        d.n_pipes = P
        d.pipe_names = self._names
        d.pipe_name_off = _ptr(self.pipe_name_off, C.c_int32)
        d.latency = _ptr(self.latency, C.c_double)
        d.latency_ok = _ptr(self.latency_ok, C.c_uint8)
        d.has_spec = _ptr(self.has_spec, C.c_uint8)
        d.model_params = _ptr(self.params, C.c_double)
        d.peak_flops = _ptr(self.peak, C.c_double)
        d.prefill_mfu = _ptr(self.mfu, C.c_double)
        d.n_workers = len(self.workers)
        d.worker_ids = _ptr(self.worker_ids, C.c_int32)
        d.headroom = instance.headroom
        d.realloc_penalty = instance.realloc_penalty
        d.default_migration_cost = instance.default_migration_cost
        d.merge_enabled = 1 if instance.merge_enabled else 0
        d.lut = _ptr(self.lut, C.c_double)
        d.alloc_sm = _ptr(self.alloc_sm, C.c_double)
        d.alloc_mem = _ptr(self.alloc_mem, C.c_double)
        self.desc = d


class GraphEncoding:
    """The static sub-stage graph of an instance (include/rlx.h
    RlxGraphDesc): every graph's nodes in Instance.graphs order, then node
    insertion order — the reference ExecState's dict order
    (scheduler.py:348-356)."""

    def __init__(self, instance, enc: "InstanceEncoding"):
        nodes = [n for g in instance.graphs for n in g.nodes.values()]
        self.ids = [n.id for n in nodes]
        self.index = {nid: i for i, nid in enumerate(self.ids)}
        self.pipe = np.array([enc.pipe_index[n.pipeline_id] for n in nodes], dtype=np.int32)
        self.worker = np.array([enc.worker_index[n.worker_id] for n in nodes], dtype=np.int32)
        self.kind = np.array([KIND_CODE[n.kind] for n in nodes], dtype=np.int32)
        self.duration = np.array([n.duration for n in nodes], dtype=np.float64)
        self.mem = np.array([n.mem_fraction for n in nodes], dtype=np.float64)
        self.remaining = np.array([n.remaining_decode_tokens for n in nodes], dtype=np.int64)
        self.active = np.array([n.active_requests for n in nodes], dtype=np.int64)
        self.context = np.array([n.context_tokens for n in nodes], dtype=np.int64)
        self.token_total = np.array([n.token_total for n in nodes], dtype=np.int64)
        self.span_lo = np.array([n.step_span[0] for n in nodes], dtype=np.int64)
        self.span_hi = np.array([n.step_span[1] for n in nodes], dtype=np.int64)
        blob = bytearray()
        offs = np.zeros(len(nodes), dtype=np.int32)
        for i, nid in enumerate(self.ids):
            offs[i] = len(blob)
            blob += nid.encode("utf-8") + b"\0"
        self._ids = bytes(blob)
        self.id_off = offs
        src, dst = [], []
        for g in instance.graphs:
            for a, b in g.edges:
                src.append(self.index[a])
                dst.append(self.index[b])
        self.edge_src = np.array(src, dtype=np.int32)
        self.edge_dst = np.array(dst, dtype=np.int32)
        d = abi.RlxGraphDesc()
        d.n_nodes = len(nodes)
        d.n_edges = len(src)
        d.pipe = _ptr(self.pipe, C.c_int32)
        d.worker = _ptr(self.worker, C.c_int32)
        d.kind = _ptr(self.kind, C.c_int32)
        d.duration = _ptr(self.duration, C.c_double)
        d.mem = _ptr(self.mem, C.c_double)
        d.remaining = _ptr(self.remaining, C.c_int64)
        d.active = _ptr(self.active, C.c_int64)
        d.context = _ptr(self.context, C.c_int64)
        d.token_total = _ptr(self.token_total, C.c_int64)
        d.span_lo = _ptr(self.span_lo, C.c_int64)
        d.span_hi = _ptr(self.span_hi, C.c_int64)
        d.ids = self._ids
        d.id_off = _ptr(self.id_off, C.c_int32)
        d.edge_src = _ptr(self.edge_src, C.c_int32)
        d.edge_dst = _ptr(self.edge_dst, C.c_int32)
        self.desc = d


def _knobs(instance) -> tuple:
    return (instance.headroom, instance.realloc_penalty, instance.default_migration_cost, instance.merge_enabled,
            len(instance.graphs))


def instance_encoding(instance) -> "InstanceEncoding":
    """The instance's C-ABI encoding, built once per Instance object (and
    rebuilt if its knobs are changed afterwards)."""
    cached = instance.__dict__.get("_rlx_encoding")
    # the model and graph list are compared by identity, holding references
    # (an id() key could be reused by a new object after the old one is freed)
    if (cached is not None and cached[0] == _knobs(instance) and cached[2] is instance.model
            and cached[3] is instance.graphs):
        return cached[1]
    enc = InstanceEncoding(instance)
    enc.graph = GraphEncoding(instance, enc)
    instance.__dict__["_rlx_encoding"] = (_knobs(instance), enc, instance.model, instance.graphs)
    return enc
