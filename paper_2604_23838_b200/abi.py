"""ctypes mirror of include/rlx.h (the C-ABI boundary)."""

from __future__ import annotations

import ctypes as C

RLX_ABI_VERSION = 4
RLX_F_NO_SYNC_STATS = 1
RLX_F_REUSE_PLAN = 2
RLX_F_SHARD = 4
RLX_NKIND = 7
RLX_NALLOC = 25
RLX_NPARTNER = 8
RLX_MAX_MEMBERS = 64

RLX_OK, RLX_ERR_ARG, RLX_ERR_CUDA, RLX_ERR_SCHEDULING, RLX_ERR_KEY, RLX_ERR_LIMIT, RLX_ERR_VALUE = range(7)
CLASS_MULTIPLEX, CLASS_MERGE, CLASS_EXCLUSIVE = 0, 1, 2

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_bp = C.POINTER(C.c_uint8)


class RlxInstanceDesc(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32), ("n_pipes", C.c_int32),
        ("pipe_names", C.c_char_p), ("pipe_name_off", _ip),
        ("latency", _dp), ("latency_ok", _bp), ("has_spec", _bp),
        ("model_params", _dp), ("peak_flops", _dp), ("prefill_mfu", _dp),
        ("n_workers", C.c_int32), ("worker_ids", _ip),
        ("headroom", C.c_double), ("realloc_penalty", C.c_double), ("default_migration_cost", C.c_double),
        ("merge_enabled", C.c_int32), ("_pad", C.c_int32),
        ("lut", _dp), ("alloc_sm", _dp), ("alloc_mem", _dp),
    ]


class RlxStateDesc(C.Structure):
    _fields_ = [
        ("now", C.c_double), ("n_nodes", C.c_int32), ("n_edges", C.c_int32),
        ("pipe", _ip), ("worker", _ip), ("kind", _ip), ("duration", _dp), ("mem", _dp),
        ("remaining", _lp), ("active", _lp), ("context", _lp), ("completed", _bp), ("merge_prefix", _dp),
        ("ids", C.c_char_p), ("id_off", _ip), ("edge_src", _ip), ("edge_dst", _ip),
        ("n_running", C.c_int32), ("n_toolwaits", C.c_int32),
        ("run_node", _ip), ("run_partner", _ip), ("run_rate", _dp), ("run_prefix", _dp), ("run_work", _dp),
        ("tw_node", _ip), ("tw_end", _dp),
        ("n_grants", C.c_int32), ("_pad", C.c_int32),
        ("grant_worker", _ip), ("grant_pipe", _ip), ("grant_mem", _dp),
    ]


class RlxDecideArgs(C.Structure):
    _fields_ = [
        ("window", C.c_int32), ("max_merge", C.c_int32),
        ("serial_begin", C.c_int64), ("serial_end", C.c_int64),
        ("keys_out", _dp), ("dev_key_out", C.c_void_p),
        ("flags", C.c_int32), ("_pad", C.c_int32),
    ]


class RlxKey(C.Structure):
    _fields_ = [("cost_bits", C.c_uint64), ("finish_bits", C.c_uint64), ("prio_serial", C.c_uint64),
                ("valid", C.c_uint64)]


class RlxAction(C.Structure):
    _fields_ = [("cls", C.c_int32), ("node_a", C.c_int32), ("node_b", C.c_int32), ("alloc", C.c_int32),
                ("target_worker", C.c_int32), ("n_members", C.c_int32),
                ("members", C.c_int32 * RLX_MAX_MEMBERS)]


class RlxDecision(C.Structure):
    _fields_ = [
        ("n_candidates", C.c_int64), ("found", C.c_int32), ("priority", C.c_int32), ("serial", C.c_int64),
        ("cost", C.c_double), ("finish", C.c_double), ("action", RlxAction), ("key", RlxKey),
        ("passes", C.c_int64), ("alg_bytes", C.c_double), ("kernel_ms", C.c_double), ("plan_ms", C.c_double),
        ("n_merge", C.c_int64), ("n_multiplex", C.c_int64), ("n_exclusive", C.c_int64),
        ("device_ms", C.c_double), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
        ("shard_begin", C.c_int64), ("shard_end", C.c_int64), ("events", C.c_int64), ("err_key", C.c_int64),
    ]


class RlxGraphDesc(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32), ("n_edges", C.c_int32),
        ("pipe", _ip), ("worker", _ip), ("kind", _ip), ("duration", _dp), ("mem", _dp),
        ("remaining", _lp), ("active", _lp), ("context", _lp), ("token_total", _lp),
        ("span_lo", _lp), ("span_hi", _lp), ("ids", C.c_char_p), ("id_off", _ip),
        ("edge_src", _ip), ("edge_dst", _ip),
    ]


class RlxApply(C.Structure):
    _fields_ = [
        ("cls", C.c_int32), ("node_a", C.c_int32), ("node_b", C.c_int32), ("target_worker", C.c_int32),
        ("n_members", C.c_int32), ("_pad", C.c_int32), ("members", C.c_int32 * RLX_MAX_MEMBERS),
        ("rate_a", C.c_double), ("rate_b", C.c_double),
        ("sm_a", C.c_double), ("mem_a", C.c_double), ("sm_b", C.c_double), ("mem_b", C.c_double),
    ]


class RlxStateInfo(C.Structure):
    _fields_ = [
        ("now", C.c_double), ("makespan", C.c_double),
        ("n_total", C.c_int32), ("n_alive", C.c_int32), ("n_done", C.c_int32), ("done", C.c_int32),
        ("has_events", C.c_int32), ("n_running", C.c_int32), ("n_toolwaits", C.c_int32), ("_pad", C.c_int32),
        ("revision", C.c_int64), ("n_events", C.c_int64),
    ]


class RlxNodeInfo(C.Structure):
    _fields_ = [
        ("pipe", C.c_int32), ("worker", C.c_int32), ("kind", C.c_int32), ("alive", C.c_int32),
        ("completed", C.c_int32), ("running", C.c_int32),
        ("duration", C.c_double), ("mem", C.c_double), ("completion_time", C.c_double),
        ("remaining", C.c_int64), ("active", C.c_int64), ("context", C.c_int64), ("token_total", C.c_int64),
        ("span_lo", C.c_int64), ("span_hi", C.c_int64), ("id", C.c_char_p),
    ]


RLX_EV_START, RLX_EV_FINISH, RLX_EV_RERATE, RLX_EV_MERGE, RLX_EV_MIGRATION, RLX_EV_TOOLWAIT_START = range(6)
EVENT_NAMES = ("start", "finish", "rerate", "merge", "migration", "toolwait-start")  # rlmux/sim.py:45


class RlxEvent(C.Structure):
    _fields_ = [("time", C.c_double), ("worker", C.c_int32), ("kind", C.c_int32), ("node", C.c_int32),
                ("_pad", C.c_int32), ("sm", C.c_double), ("mem", C.c_double)]


class RlxDriveArgs(C.Structure):
    _fields_ = [("window", C.c_int32), ("max_merge", C.c_int32), ("max_decisions", C.c_int64),
                ("max_steps", C.c_int64)]


class RlxStep(C.Structure):
    _fields_ = [("start", C.c_double), ("action", RlxAction), ("cost", C.c_double), ("finish", C.c_double),
                ("priority", C.c_int32), ("_pad", C.c_int32), ("serial", C.c_int64), ("n_candidates", C.c_int64),
                ("decision_ms", C.c_double), ("kernel_ms", C.c_double)]


class RlxPlanInfo(C.Structure):
    _fields_ = [("n_candidates", C.c_int64), ("n_multiplex", C.c_int64), ("n_merge", C.c_int64),
                ("n_exclusive", C.c_int64), ("window_nodes", C.c_int32), ("local_nodes", C.c_int32),
                ("max_worker_order", C.c_int32), ("hot_bytes", C.c_int32), ("blob_bytes", C.c_int64)]


class RlxRolloutTables(C.Structure):
    _fields_ = [("n_samples", C.c_int32), ("n_workers", C.c_int32), ("worker_of", C.POINTER(C.c_int32)),
                ("prompt", C.POINTER(C.c_int64)), ("turn_off", C.POINTER(C.c_int32)),
                ("turn_prefill", C.POINTER(C.c_int64)), ("turn_decode", C.POINTER(C.c_int64)),
                ("turn_tool", C.POINTER(C.c_double)), ("latency", C.c_double * 5)]


class RlxSegment(C.Structure):
    _fields_ = [("worker", C.c_int32), ("seq", C.c_int32), ("kind", C.c_int32), ("bucket", C.c_int32),
                ("step_lo", C.c_int64), ("step_hi", C.c_int64), ("decode", C.c_int64), ("active0", C.c_int64),
                ("context0", C.c_int64), ("tokens", C.c_int64), ("duration", C.c_double)]


class RlxSimAction(C.Structure):
    _fields_ = [("start", C.c_double), ("sm", C.c_double), ("mem", C.c_double), ("cls", C.c_int32),
                ("target_worker", C.c_int32), ("n_ids", C.c_int32), ("id_off", C.c_int32)]


class RlxSimResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("action_index", C.c_int32), ("makespan", C.c_double),
                ("throughput", C.c_double), ("total_tokens", C.c_int64), ("error", C.c_char * 192)]


# Every symbol include/rlx.h declares (checked by tests/test_abi.py).
EXPORTED = ("rlx_abi_version", "rlx_open", "rlx_load_instance", "rlx_decide", "rlx_decode",
            "rlx_last_error", "rlx_error_text", "rlx_close", "rlx_set_stream", "rlx_drive", "rlx_plan_info",
            "rlx_state_create", "rlx_state_clone", "rlx_state_destroy", "rlx_state_error", "rlx_state_apply",
            "rlx_state_advance", "rlx_state_info", "rlx_state_snapshot", "rlx_state_node", "rlx_state_events",
            "rlx_state_completion", "rlx_graph_build", "rlx_graph_segments", "rlx_graph_stats", "rlx_graph_error",
            "rlx_graph_free", "rlx_simulate_batch", "rlx_enumerate", "rlx_branch_and_bound")


def bind(lib: C.CDLL) -> C.CDLL:
    lib.rlx_abi_version.restype = C.c_int
    lib.rlx_abi_version.argtypes = []
    lib.rlx_open.restype = C.c_int
    lib.rlx_open.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.rlx_load_instance.restype = C.c_int
    lib.rlx_load_instance.argtypes = [C.c_void_p, C.POINTER(RlxInstanceDesc)]
    lib.rlx_decide.restype = C.c_int
    lib.rlx_decide.argtypes = [C.c_void_p, C.POINTER(RlxStateDesc), C.POINTER(RlxDecideArgs),
                               C.POINTER(RlxDecision)]
    lib.rlx_decode.restype = C.c_int
    lib.rlx_decode.argtypes = [C.c_void_p, C.c_int64, C.POINTER(RlxAction)]
    lib.rlx_last_error.restype = C.c_char_p
    lib.rlx_last_error.argtypes = [C.c_void_p]
    lib.rlx_error_text.restype = C.c_int
    lib.rlx_error_text.argtypes = [C.c_int32, C.c_char_p, C.c_int32]
    lib.rlx_set_stream.restype = C.c_int
    lib.rlx_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    lib.rlx_close.restype = None
    lib.rlx_close.argtypes = [C.c_void_p]
    lib.rlx_drive.restype = C.c_int
    lib.rlx_drive.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(RlxDriveArgs), C.POINTER(RlxStep),
                              C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.rlx_plan_info.restype = C.c_int
    lib.rlx_plan_info.argtypes = [C.POINTER(RlxInstanceDesc), C.POINTER(RlxStateDesc), C.c_int32, C.c_int32,
                                  C.POINTER(RlxPlanInfo), C.c_char_p, C.c_int32]
    lib.rlx_state_create.restype = C.c_int
    lib.rlx_state_create.argtypes = [C.POINTER(RlxInstanceDesc), C.POINTER(RlxGraphDesc), C.c_int,
                                     C.POINTER(C.c_void_p)]
    lib.rlx_state_clone.restype = C.c_int
    lib.rlx_state_clone.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    lib.rlx_state_destroy.restype = None
    lib.rlx_state_destroy.argtypes = [C.c_void_p]
    lib.rlx_state_error.restype = C.c_char_p
    lib.rlx_state_error.argtypes = [C.c_void_p]
    lib.rlx_state_apply.restype = C.c_int
    lib.rlx_state_apply.argtypes = [C.c_void_p, C.POINTER(RlxApply)]
    lib.rlx_state_advance.restype = C.c_int
    lib.rlx_state_advance.argtypes = [C.c_void_p, C.c_int, C.c_double]
    lib.rlx_state_info.restype = C.c_int
    lib.rlx_state_info.argtypes = [C.c_void_p, C.POINTER(RlxStateInfo)]
    lib.rlx_state_snapshot.restype = C.c_int
    lib.rlx_state_snapshot.argtypes = [C.c_void_p, C.POINTER(RlxStateDesc)]
    lib.rlx_state_node.restype = C.c_int
    lib.rlx_state_node.argtypes = [C.c_void_p, C.c_int32, C.POINTER(RlxNodeInfo)]
    lib.rlx_state_events.restype = C.c_int
    lib.rlx_state_events.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(RlxEvent)]
    lib.rlx_graph_build.restype = C.c_int
    lib.rlx_graph_build.argtypes = [C.c_int, C.c_int32, C.POINTER(RlxRolloutTables), C.POINTER(C.c_int32), C.c_int32,
                                    C.c_int32, C.POINTER(C.c_void_p)]
    lib.rlx_graph_segments.restype = C.c_int
    lib.rlx_graph_segments.argtypes = [C.c_void_p, C.c_int32, C.POINTER(RlxSegment), C.c_int64, C.POINTER(C.c_int64)]
    lib.rlx_graph_stats.restype = C.c_int
    lib.rlx_graph_stats.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    lib.rlx_graph_error.restype = C.c_char_p
    lib.rlx_graph_error.argtypes = [C.c_void_p]
    lib.rlx_graph_free.restype = None
    lib.rlx_graph_free.argtypes = [C.c_void_p]
    lib.rlx_simulate_batch.restype = C.c_int
    lib.rlx_simulate_batch.argtypes = [C.POINTER(RlxInstanceDesc), C.POINTER(RlxGraphDesc), C.c_int32,
                                       C.POINTER(C.c_int64), C.POINTER(RlxSimAction), C.c_char_p, C.c_int32,
                                       C.POINTER(RlxSimResult), C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_double)]
    lib.rlx_enumerate.restype = C.c_int
    lib.rlx_enumerate.argtypes = [C.POINTER(RlxInstanceDesc), C.c_void_p, C.POINTER(RlxAction), C.c_int64,
                                  C.POINTER(C.c_int64)]
    lib.rlx_branch_and_bound.restype = C.c_int
    lib.rlx_branch_and_bound.argtypes = [C.POINTER(RlxInstanceDesc), C.POINTER(RlxGraphDesc), C.c_double, C.c_int32,
                                         C.POINTER(RlxStep), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int64)]
    lib.rlx_state_completion.restype = C.c_int
    lib.rlx_state_completion.argtypes = [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_double)]
    return lib
