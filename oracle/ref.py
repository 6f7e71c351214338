"""TEST INFRASTRUCTURE ONLY — ctypes driver for the reference oracle.

Loads oracle/_ref/libref_shim.so (the UNMODIFIED reference collsight library
compiled from /root/reference/proj/src by oracle/Makefile, plus the thin
adapter oracle/ref_shim.cpp) and exposes the reference's C++ analyzer entry
points on the same packed records and tables the B200 engine consumes.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module, and only as the checker / the timed CPU reference.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import List, Optional, Tuple

import numpy as np

from paper_2509_03018_b200 import _abi
from paper_2509_03018_b200.model import (AnalysisConfig, Topology, OpProgram,
                                         TriggerConfig, TriggerEvent,
                                         layout_from_json)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libref_shim.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_trigger_state_new.restype = C.c_void_p
        _lib.ref_trigger_state_free.argtypes = [C.c_void_p]
        _lib.ref_free.argtypes = [C.c_void_p]
    return _lib


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.msg = msg


def _check(st):
    if st != 0:
        raise RefError(st, lib().ref_last_error().decode())


def _take(p: C.c_void_p) -> str:
    if not p.value:
        return ""
    s = C.string_at(p.value).decode()
    lib().ref_free(p)
    return s


def _recs(recs: np.ndarray):
    recs = np.ascontiguousarray(recs, dtype=_abi.RECORD_DTYPE)
    return recs, _abi.ptr(recs), C.c_size_t(len(recs))


def simulate(cfg_json: str, with_jsonl: bool = False):
    out = C.c_void_p()
    n = C.c_size_t()
    jl = C.c_void_p()
    _check(lib().ref_simulate(cfg_json.encode(), C.byref(out), C.byref(n),
                              C.byref(jl) if with_jsonl else None))
    arr = np.frombuffer(C.string_at(out.value, n.value * 48),
                        dtype=_abi.RECORD_DTYPE).copy() if n.value else \
        np.zeros(0, dtype=_abi.RECORD_DTYPE)
    lib().ref_free(out)
    return (arr, _take(jl)) if with_jsonl else arr


def simulate_prog(cfg_json: str, prog: OpProgram, msg_bytes: int) -> np.ndarray:
    """Reference run_simulation with a custom program;
    layout, sim config and faults from the scenario JSON."""
    out = C.c_void_p()
    n = C.c_size_t()
    pd, keep = prog.desc()
    _check(lib().ref_simulate_prog(cfg_json.encode(), C.byref(pd),
                                   C.c_uint64(msg_bytes), C.byref(out), C.byref(n)))
    arr = np.frombuffer(C.string_at(out.value, n.value * 48),
                        dtype=_abi.RECORD_DTYPE).copy() if n.value else \
        np.zeros(0, dtype=_abi.RECORD_DTYPE)
    lib().ref_free(out)
    return arr


def run_detection_cfg(cfg_json: str, recs: np.ndarray):
    """-> (reports_to_jsonl text, full reports list, sampled, seconds)"""
    recs, p, n = _recs(recs)
    rep = C.c_void_p()
    full = C.c_void_p()
    sampled = np.zeros(1 << 16, dtype=np.int32)
    ns = C.c_size_t()
    secs = C.c_double()
    _check(lib().ref_run_detection_cfg(cfg_json.encode(), p, n, C.byref(rep),
                                       C.byref(full), _abi.ptr(sampled),
                                       C.c_size_t(len(sampled)), C.byref(ns),
                                       C.byref(secs)))
    return (_take(rep), [json.loads(l) for l in _take(full).splitlines()],
            sampled[: ns.value].tolist(), secs.value)


def run_detection(topo: Topology, prog: OpProgram, tcfg: TriggerConfig,
                  acfg: AnalysisConfig, seed: int, recs: np.ndarray,
                  onset: Optional[float] = None):
    recs, p, n = _recs(recs)
    td, k1 = topo.desc()
    pd, k2 = prog.desc()
    tc, ac = tcfg.c(), acfg.c()
    rep = C.c_void_p()
    full = C.c_void_p()
    secs = C.c_double()
    _check(lib().ref_run_detection(C.byref(td), C.byref(pd), C.byref(tc),
                                   C.byref(ac), C.c_uint64(seed), p, n,
                                   C.c_int(onset is not None),
                                   C.c_double(onset or 0.0), C.byref(rep),
                                   C.byref(full), C.byref(secs)))
    return (_take(rep), [json.loads(l) for l in _take(full).splitlines()],
            secs.value)


def analyze(topo: Topology, prog: OpProgram, acfg: AnalysisConfig,
            recs: np.ndarray, trigger: TriggerEvent, mode: int = 0):
    recs, p, n = _recs(recs)
    td, k1 = topo.desc()
    pd, k2 = prog.desc()
    ac = acfg.c()
    tr = trigger.c()
    full = C.c_void_p()
    secs = C.c_double()
    _check(lib().ref_analyze(C.byref(td), C.byref(pd), C.byref(ac), p, n,
                             C.byref(tr), C.c_int(mode), C.byref(full),
                             C.byref(secs)))
    return json.loads(_take(full))


def affected_groups(topo, prog, acfg, recs, trigger) -> Tuple[List[int], int]:
    recs, p, n = _recs(recs)
    td, k1 = topo.desc()
    pd, k2 = prog.desc()
    ac = acfg.c()
    tr = trigger.c()
    out = np.zeros(max(1, len(topo.groups)), dtype=np.int32)
    no = C.c_size_t()
    sc = C.c_uint64()
    _check(lib().ref_affected_groups(C.byref(td), C.byref(pd), C.byref(ac), p,
                                     n, C.byref(tr), _abi.ptr(out),
                                     C.c_size_t(len(out)), C.byref(no),
                                     C.byref(sc)))
    return out[: no.value].tolist(), sc.value


def query(recs, ranks, t0, t1) -> List[int]:
    recs, p, n = _recs(recs)
    r = np.ascontiguousarray(ranks, dtype=np.int32)
    out = np.zeros(max(1, len(recs)), dtype=np.uint64)
    no = C.c_size_t()
    _check(lib().ref_query(p, n, _abi.ptr(r), C.c_size_t(len(r)),
                           C.c_double(t0), C.c_double(t1), _abi.ptr(out),
                           C.c_size_t(len(out)), C.byref(no)))
    return out[: no.value].tolist()


def last_log_per_rank(recs, members, t):
    recs, p, n = _recs(recs)
    m = np.ascontiguousarray(members, dtype=np.int32)
    orank = np.zeros(max(1, len(m)), dtype=np.int32)
    oidx = np.zeros(max(1, len(m)), dtype=np.uint64)
    no = C.c_size_t()
    _check(lib().ref_last_log_per_rank(p, n, _abi.ptr(m), C.c_size_t(len(m)),
                                       C.c_double(t), _abi.ptr(orank),
                                       _abi.ptr(oidx), C.byref(no)))
    return list(zip(orank[: no.value].tolist(), oidx[: no.value].tolist()))


class TriggerState:
    def __init__(self):
        self.h = C.c_void_p(lib().ref_trigger_state_new())

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_trigger_state_free(self.h)
            self.h = None


def evaluate(recs, sampled, t, state: TriggerState, cfg: TriggerConfig):
    recs, p, n = _recs(recs)
    s = np.ascontiguousarray(sampled, dtype=np.int32)
    tripped = C.c_int()
    ev = _abi.TriggerEventC()
    tc = cfg.c()
    _check(lib().ref_evaluate(p, n, _abi.ptr(s), C.c_size_t(len(s)),
                              C.c_double(t), state.h, C.byref(tc),
                              C.byref(tripped), C.byref(ev)))
    if not tripped.value:
        return None
    return TriggerEvent(ev.kind, ev.suspect_rank, ev.time_ms)


def sample_ranks(topo: Topology, max_sampled: int, seed: int) -> List[int]:
    td, k = topo.desc()
    out = np.zeros(max(1, len(topo.groups) + 1), dtype=np.int32)
    no = C.c_size_t()
    _check(lib().ref_sample_ranks(C.byref(td), C.c_int32(max_sampled),
                                  C.c_uint64(seed), _abi.ptr(out),
                                  C.c_size_t(len(out)), C.byref(no)))
    return out[: no.value].tolist()


def layout(tp, pp, dp, rpn, cpp, nics=4, msg_bytes=1 << 26):
    js = C.c_void_p()
    _check(lib().ref_layout(tp, pp, dp, rpn, cpp, nics, C.c_uint64(msg_bytes),
                            C.byref(js)))
    return layout_from_json(_take(js), tp, pp, dp)


def check_min_op(pairs):
    r = np.array([a for a, _ in pairs], dtype=np.int32)
    o = np.array([b for _, b in pairs], dtype=np.int64)
    out = np.zeros(max(1, len(pairs)), dtype=np.int32)
    no = C.c_size_t()
    has = C.c_int()
    _check(lib().ref_check_min_op(_abi.ptr(r), _abi.ptr(o), C.c_size_t(len(r)),
                                  _abi.ptr(out), C.byref(no), C.byref(has)))
    return out[: no.value].tolist() if has.value else None


def check_min_data(pairs):
    r = np.array([a for a, _ in pairs], dtype=np.int32)
    pr = (_abi.ProgressC * max(1, len(pairs)))()
    for i, (_, t) in enumerate(pairs):
        pr[i] = _abi.ProgressC(*t)
    out = np.zeros(max(1, len(pairs)), dtype=np.int32)
    no = C.c_size_t()
    _check(lib().ref_check_min_data(_abi.ptr(r), pr, C.c_size_t(len(r)),
                                    _abi.ptr(out), C.byref(no)))
    return out[: no.value].tolist()


def check_rc_table(c, peer=None):
    a = _abi.ProgressC(*c)
    b = _abi.ProgressC(*peer) if peer is not None else None
    cat = C.c_int()
    side = C.c_int()
    _check(lib().ref_check_rc_table(C.byref(a), C.byref(b) if b else None,
                                    C.byref(cat), C.byref(side)))
    return cat.value, side.value


class RefStore:
    """A reference TraceStore built once in this process (CPU leg of bench)."""

    def __init__(self, recs: np.ndarray):
        recs, p, n = _recs(recs)
        lib().ref_store_new.restype = C.c_void_p
        self.h = C.c_void_p(lib().ref_store_new(p, n))
        self.n = len(recs)

    def window(self, cfg_json: str, t: float):
        """-> (evaluate seconds, analyze seconds, tripped, full report or None)"""
        e = C.c_double()
        a = C.c_double()
        tr = C.c_int()
        full = C.c_void_p()
        _check(lib().ref_window(self.h, cfg_json.encode(), C.c_double(t), C.byref(e),
                                C.byref(a), C.byref(tr), C.byref(full)))
        rep = json.loads(_take(full)) if tr.value else None
        return e.value, a.value, bool(tr.value), rep

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            lib().ref_store_free.argtypes = [C.c_void_p]
            lib().ref_store_free(self.h)
            self.h = None
