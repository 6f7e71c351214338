"""ctypes / numpy mirrors of the plain-C structs in include/csg_engine.h.

Pure layout definitions (no compute); shared by the host mirror and the test
oracle so both hand byte-identical inputs to their libraries.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

# csg_packed_record (48 bytes). The union payload is exposed through
# overlapping fields: completions use start_ms/msg_bytes, states use the
# three u32 counters. Mirrors CompletionRecord/StateRecord
# (reference proj/include/collsight/trace.hpp:19-46).
RECORD_DTYPE = np.dtype(
    {
        "names": [
            "ts", "op_seq", "rank", "comm_id", "channel", "kind", "op_name",
            "reserved", "start_ms", "msg_bytes", "gpu_ready",
            "rdma_transmitted", "rdma_done", "s_reserved",
        ],
        "formats": [
            "<f8", "<i8", "<i4", "<i4", "<i4", "u1", "u1", "<u2", "<f8",
            "<u8", "<u4", "<u4", "<u4", "<u4",
        ],
        "offsets": [0, 8, 16, 20, 24, 28, 29, 30, 32, 40, 32, 36, 40, 44],
        "itemsize": 48,
    }
)
assert RECORD_DTYPE.itemsize == 48

KIND_COMPLETION, KIND_STATE = 0, 1
OP_NAMES = ["AllGather", "ReduceScatter", "AllReduce", "Send", "Recv"]
OP_ALLGATHER, OP_REDUCESCATTER, OP_ALLREDUCE, OP_SEND, OP_RECV = range(5)
GROUP_KINDS = ["DP", "PP", "TP"]
TRIGGER_KINDS = ["failure", "straggler"]
RC_CATEGORIES = [
    "uninitialized_or_blocked",
    "rdma_issue_or_receiver_not_ready",
    "rdma_issue_or_receiver_failed",
    "gpu_issue",
    "straggler_late_start",
    "straggler_late_end",
    "flow_incomplete",
    "flow_skewed",
]
SIDES = ["local", "remote", "undetermined"]
VERDICTS = ["suspects", "undetermined", "false_trigger", "insufficient_history",
            "no_straggler"]


class TopologyDesc(C.Structure):
    _fields_ = [
        ("world_size", C.c_int32),
        ("n_groups", C.c_int32),
        ("group_kind", C.c_void_p),
        ("member_off", C.c_void_p),
        ("members", C.c_void_p),
    ]


class ProgramDesc(C.Structure):
    _fields_ = [
        ("n_ops", C.c_int32),
        ("op_name", C.c_void_p),
        ("group", C.c_void_p),
        ("src", C.c_void_p),
        ("dst", C.c_void_p),
        ("dep_off", C.c_void_p),
        ("deps", C.c_void_p),
    ]


class TriggerConfigC(C.Structure):
    _fields_ = [
        ("delta_ms", C.c_double),
        ("detect_interval_ms", C.c_double),
        ("throughput_drop_factor", C.c_double),
        ("interval_inflation_factor", C.c_double),
        ("max_sampled_ranks", C.c_int32),
        ("warmup_windows", C.c_int32),
        ("ema_alpha", C.c_double),
    ]


class AnalysisConfigC(C.Structure):
    _fields_ = [
        ("straggler_threshold_ms", C.c_double),
        ("delta_ms", C.c_double),
        ("flow_skew_factor", C.c_double),
        ("consecutive_iterations_k", C.c_int32),
        ("reserved", C.c_int32),
    ]


class TriggerEventC(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("suspect_rank", C.c_int32),
        ("time_ms", C.c_double),
    ]


class SuspectC(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("category", C.c_uint8),
        ("side", C.c_uint8),
        ("reserved", C.c_uint16),
        ("group", C.c_int32),
        ("reserved2", C.c_int32),
        ("stuck_op", C.c_int64),
        ("onset_ms", C.c_double),
    ]


class EvidenceC(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("channel", C.c_int32),
        ("time_ms", C.c_double),
        ("op_seq", C.c_int64),
    ]


class ReportViewC(C.Structure):
    _fields_ = [
        ("verdict", C.c_int32),
        ("trigger", TriggerEventC),
        ("suspects", C.POINTER(SuspectC)),
        ("n_suspects", C.c_size_t),
        ("exonerated", C.POINTER(SuspectC)),
        ("n_exonerated", C.c_size_t),
        ("affected_groups", C.POINTER(C.c_int32)),
        ("n_affected", C.c_size_t),
        ("evidence", C.POINTER(EvidenceC)),
        ("n_evidence", C.c_size_t),
        ("records_scanned", C.c_uint64),
    ]


class ProgressC(C.Structure):
    _fields_ = [
        ("gpu_ready", C.c_uint64),
        ("rdma_transmitted", C.c_uint64),
        ("rdma_done", C.c_uint64),
    ]


def ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)
