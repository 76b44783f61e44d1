"""Instance / state -> the flat arrays of the C-ABI (include/rlx.h).

`InstanceEncoding` is built once per instance: pipeline table, knobs and
the slowdown LUT. The LUT holds every factor the chooser can query —
FULL_ALLOCATION, the 12 Multiplex allocations (MUX_SM_GRID x MEM_GRID,
rlmux/scheduler.py:671-675) and their complements (slowdown.py:169-175) —
for all (kind, partner) pairs, evaluated here with the reference's own
bilinear op order so the device only does table lookups.

`StateEncoding` is a snapshot of `HostState` at a decision point. Node
arrays are cached per structural revision (merges change the graph), so an
undisturbed decision only refreshes the dynamic vectors.
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


class StateEncoding:
    """Flat snapshot of a HostState (scheduler.py:339-366 fields)."""

    def __init__(self, enc: InstanceEncoding):
        self.enc = enc
        self._rev = None

    def _structure(self, st):
        enc = self.enc
        order = list(st.nodes)
        self.order = order
        self.index = {nid: i for i, nid in enumerate(order)}
        n = len(order)
        nodes = [st.nodes[k] for k in order]
        self.pipe = np.array([enc.pipe_index[x.pipeline_id] for x in nodes], dtype=np.int32)
        self.worker = np.array([enc.worker_index[x.worker_id] for x in nodes], dtype=np.int32)
        self.kind = np.array([KIND_CODE[x.kind] for x in nodes], dtype=np.int32)
        self.duration = np.array([x.duration for x in nodes], dtype=np.float64)
        self.mem = np.array([x.mem_fraction for x in nodes], dtype=np.float64)
        self.remaining = np.array([x.remaining_decode_tokens for x in nodes], dtype=np.int64)
        self.active = np.array([x.active_requests for x in nodes], dtype=np.int64)
        self.context = np.array([x.context_tokens for x in nodes], dtype=np.int64)
        blob = bytearray()
        offs = np.zeros(n, dtype=np.int32)
        for i, k in enumerate(order):
            offs[i] = len(blob)
            blob += k.encode("utf-8") + b"\0"
        self._ids = bytes(blob)
        self.id_off = offs
        src, dst = [], []
        idx = self.index
        for k in order:
            i = idx[k]
            for s in st.succs[k]:
                src.append(i)
                dst.append(idx[s])
        self.edge_src = np.array(src, dtype=np.int32)
        self.edge_dst = np.array(dst, dtype=np.int32)
        self._rev = (id(st), st.revision)

    def encode(self, st):
        if self._rev != (id(st), st.revision):
            self._structure(st)
        enc = self.enc
        idx = self.index
        n = len(self.order)
        self.completed = np.zeros(n, dtype=np.uint8)
        for k in st.completed:
            self.completed[idx[k]] = 1
        self.merge_prefix = np.zeros(n, dtype=np.float64)
        for k, v in st.merge_prefix.items():
            i = idx.get(k)  # a merged node merged again leaves a dead entry (reference quirk)
            if i is not None:
                self.merge_prefix[i] = v
        run = list(st.running.items())
        self.run_node = np.array([idx[k] for k, _ in run], dtype=np.int32)
        self.run_partner = np.array([idx[m.partner_id] if m.partner_id is not None else -1 for _, m in run],
                                    dtype=np.int32)
        self.run_rate = np.array([m.rate for _, m in run], dtype=np.float64)
        self.run_prefix = np.array([m.prefix_left for _, m in run], dtype=np.float64)
        self.run_work = np.array([m.work_left for _, m in run], dtype=np.float64)
        tws = list(st.toolwaits.items())
        self.tw_node = np.array([idx[k] for k, _ in tws], dtype=np.int32)
        self.tw_end = np.array([t for _, t in tws], dtype=np.float64)
        grants = list(st.last_mem_grant.items())
        self.grant_worker = np.array([enc.worker_index[w] for (w, _), _ in grants], dtype=np.int32)
        self.grant_pipe = np.array([enc.pipe_index[p] for (_, p), _ in grants], dtype=np.int32)
        self.grant_mem = np.array([m for _, m in grants], dtype=np.float64)
        d = abi.RlxStateDesc()
        d.now = st.now
        d.n_nodes = n
        d.n_edges = len(self.edge_src)
        d.pipe = _ptr(self.pipe, C.c_int32)
        d.worker = _ptr(self.worker, C.c_int32)
        d.kind = _ptr(self.kind, C.c_int32)
        d.duration = _ptr(self.duration, C.c_double)
        d.mem = _ptr(self.mem, C.c_double)
        d.remaining = _ptr(self.remaining, C.c_int64)
        d.active = _ptr(self.active, C.c_int64)
        d.context = _ptr(self.context, C.c_int64)
        d.completed = _ptr(self.completed, C.c_uint8)
        d.merge_prefix = _ptr(self.merge_prefix, C.c_double)
        d.ids = self._ids
        d.id_off = _ptr(self.id_off, C.c_int32)
        d.edge_src = _ptr(self.edge_src, C.c_int32)
        d.edge_dst = _ptr(self.edge_dst, C.c_int32)
        d.n_running = len(run)
        d.n_toolwaits = len(tws)
        d.run_node = _ptr(self.run_node, C.c_int32)
        d.run_partner = _ptr(self.run_partner, C.c_int32)
        d.run_rate = _ptr(self.run_rate, C.c_double)
        d.run_prefix = _ptr(self.run_prefix, C.c_double)
        d.run_work = _ptr(self.run_work, C.c_double)
        d.tw_node = _ptr(self.tw_node, C.c_int32)
        d.tw_end = _ptr(self.tw_end, C.c_double)
        d.n_grants = len(grants)
        d.grant_worker = _ptr(self.grant_worker, C.c_int32)
        d.grant_pipe = _ptr(self.grant_pipe, C.c_int32)
        d.grant_mem = _ptr(self.grant_mem, C.c_double)
        # the descriptor owns the arrays it points into, so it stays valid
        # after a later encode() rebinds the attributes above
        d._keep = (self.pipe, self.worker, self.kind, self.duration, self.mem, self.remaining, self.active,
                   self.context, self.completed, self.merge_prefix, self._ids, self.id_off, self.edge_src,
                   self.edge_dst, self.run_node, self.run_partner, self.run_rate, self.run_prefix, self.run_work,
                   self.tw_node, self.tw_end, self.grant_worker, self.grant_pipe, self.grant_mem)
        self.desc = d
        return d

    def action_from_raw(self, a: abi.RlxAction):
        """Decoded RlxAction -> Exclusive / Multiplex / Merge of this package."""
        from .model import Exclusive, Merge, Multiplex

        order = self.order
        if a.cls == abi.CLASS_EXCLUSIVE:
            return Exclusive(order[a.node_a])
        if a.cls == abi.CLASS_MULTIPLEX:
            return Multiplex(order[a.node_a], order[a.node_b], self.enc.allocs[a.alloc])
        ids = tuple(order[a.members[i]] for i in range(a.n_members))
        return Merge(ids, self.enc.workers[a.target_worker])
