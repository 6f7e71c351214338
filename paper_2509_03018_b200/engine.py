"""Python host mirror of the collsight analyzer API over the B200 engine.

Same entry points and argument meaning as the reference's C++ API
(proj/include/collsight/{trace,trigger,rca,runner}.hpp) and C API
(proj/include/collsight/collsight.h), bound with ctypes to the in-tree
libcollsight_b200.so (include/csg_engine.h, include/collsight.h,
include/collsight_b200.h). Every analysis call runs the sm_100a kernels;
there is no CPU fallback: importing this module on a machine without the
built library, or calling into it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .model import (AnalysisConfig, OpProgram, Topology, TriggerConfig,
                    TriggerEvent, layout_from_json)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                        "libcollsight_b200.so")

_lib = None


class EngineError(RuntimeError):
    """A non-OK csg_status / collsight_status; .status holds the code
    (2 config, 3 trace parse, 4 runtime/data, 5 argument)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status
        self.msg = msg


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`python -m paper_2509_03018_b200.build` (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.csg_last_error.restype = C.c_char_p
        L.csg_version.restype = C.c_char_p
        L.collsight_last_error.restype = C.c_char_p
        L.collsight_version.restype = C.c_char_p
        for f in ("collsight_result_text", "collsight_result_summary_json",
                  "collsight_result_reports_jsonl"):
            getattr(L, f).restype = C.c_char_p
            getattr(L, f).argtypes = [C.c_void_p]
        L.collsight_result_trigger_count.restype = C.c_uint64
        L.collsight_result_trigger_count.argtypes = [C.c_void_p]
        L.collsight_result_free.argtypes = [C.c_void_p]
        L.collsight_scenario_free.argtypes = [C.c_void_p]
        L.csg_store_size.restype = C.c_size_t
        L.csg_store_size.argtypes = [C.c_void_p]
        L.csg_results_count.restype = C.c_size_t
        L.csg_results_count.argtypes = [C.c_void_p]
        for f in ("csg_ctx_free", "csg_store_free", "csg_model_free",
                  "csg_trigger_state_free", "csg_results_free",
                  "csg_ctx_reset_stats", "collsight_b200_free"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = None
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise EngineError(st, lib().csg_last_error().decode())


def _ccheck(st: int):
    if st != 0:
        raise EngineError(st, lib().collsight_last_error().decode())


def version() -> str:
    return lib().csg_version().decode()


# ---------------------------------------------------------------------------
# Device context
# ---------------------------------------------------------------------------
class Context:
    """One CUDA device + stream (csg_ctx)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _check(lib().csg_ctx_create(C.c_int(device), C.byref(self.h)))
        self.device = device

    def stats(self) -> Tuple[float, int]:
        ms = C.c_double()
        n = C.c_uint64()
        _check(lib().csg_ctx_stats(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def reset_stats(self):
        lib().csg_ctx_reset_stats(self.h)

    def profile(self, enable: bool = True):
        _check(lib().csg_ctx_profile(self.h, C.c_int(1 if enable else 0)))

    def kernel_stats(self):
        """-> ({kernel: (total_ms, launches)}, h2d_bytes, d2h_bytes)"""
        buf = C.create_string_buffer(1 << 16)
        h2d = C.c_uint64()
        d2h = C.c_uint64()
        _check(lib().csg_ctx_kernel_stats(self.h, buf, C.c_size_t(len(buf)),
                                          C.byref(h2d), C.byref(d2h)))
        return ({k: tuple(v) for k, v in json.loads(buf.value.decode()).items()},
                h2d.value, d2h.value)

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """Join the NCCL communicator of a sharded store (csg_ctx_comm_init)."""
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id[:128])
        _check(lib().csg_ctx_comm_init(self.h, buf, C.c_size_t(128), C.c_int(nranks),
                                       C.c_int(rank)))

    def comm_info(self):
        nr = C.c_int()
        rk = C.c_int()
        coll = C.c_uint64()
        _check(lib().csg_ctx_comm_info(self.h, C.byref(nr), C.byref(rk), C.byref(coll)))
        return nr.value, rk.value, coll.value

    @classmethod
    def of_c_api(cls) -> "Context":
        """The context the collsight_* C API runs on (not owned)."""
        c = cls.__new__(cls)
        c.h = C.c_void_p()
        _ccheck(lib().collsight_b200_engine_context(C.byref(c.h)))
        c.device = -1
        c.close = lambda: None
        return c

    def close(self):
        if self.h:
            lib().csg_ctx_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("COLLSIGHT_B200_DEVICE", "0")))
    return _default_ctx


# ---------------------------------------------------------------------------
# TraceStore (proj/include/collsight/trace.hpp:101-124)
# ---------------------------------------------------------------------------
class TraceStore:
    def __init__(self, ctx: Optional[Context] = None, records: Optional[np.ndarray] = None):
        self.ctx = ctx or default_context()
        self.h = C.c_void_p()
        _check(lib().csg_store_create(self.ctx.h, C.byref(self.h)))
        if records is not None:
            self.append(records)

    def append(self, records: np.ndarray):
        r = np.ascontiguousarray(np.atleast_1d(records), dtype=_abi.RECORD_DTYPE)
        _check(lib().csg_store_append(self.h, _abi.ptr(r), C.c_size_t(len(r))))

    def append_jsonl(self, text) -> bool:
        """JSONL trace text parsed on the device (csg_store_append_jsonl).
        False: the device parser deferred (store unchanged) — parse with
        parse_trace() (the exact host parser) instead."""
        b = text.encode() if isinstance(text, str) else bytes(text)
        acc = C.c_int()
        _check(lib().csg_store_append_jsonl(self.h, b, C.c_size_t(len(b)), C.byref(acc)))
        return bool(acc.value)

    def append_jsonl_file(self, path: str) -> bool:
        acc = C.c_int()
        _check(lib().csg_store_append_jsonl_file(self.h, path.encode(), C.byref(acc)))
        return bool(acc.value)

    def records(self) -> np.ndarray:
        """The store's packed records in store order (device -> host copy)."""
        n = self.size()
        out = np.zeros(n, dtype=_abi.RECORD_DTYPE)
        if n:
            _check(lib().csg_store_records(self.h, _abi.ptr(out), C.c_size_t(n)))
        return out

    def append_device(self, ptr: int, n: int):
        _check(lib().csg_store_append_device(self.h, C.c_void_p(ptr), C.c_size_t(n)))

    def reserve(self, n: int):
        _check(lib().csg_store_reserve(self.h, C.c_size_t(n)))

    def clear(self):
        _check(lib().csg_store_clear(self.h))

    def size(self) -> int:
        return lib().csg_store_size(self.h)

    __len__ = size

    def build_index(self):
        _check(lib().csg_store_build_index(self.h))

    def invalidate(self):
        _check(lib().csg_store_invalidate(self.h))

    def query(self, ranks: Sequence[int], t0: float, t1: float) -> List[int]:
        r = np.ascontiguousarray(ranks, dtype=np.int32)
        cap = self.size() + 1
        out = np.zeros(cap, dtype=np.uint64)
        n = C.c_size_t()
        _check(lib().csg_store_query(self.h, _abi.ptr(r), C.c_size_t(len(r)),
                                     C.c_double(t0), C.c_double(t1),
                                     _abi.ptr(out), C.c_size_t(cap), C.byref(n)))
        return out[: n.value].tolist()

    def last_log_per_rank(self, members: Sequence[int], t: float):
        m = np.ascontiguousarray(members, dtype=np.int32)
        orank = np.zeros(max(1, len(m)), dtype=np.int32)
        oidx = np.zeros(max(1, len(m)), dtype=np.uint64)
        n = C.c_size_t()
        _check(lib().csg_store_last_log_per_rank(
            self.h, _abi.ptr(m), C.c_size_t(len(m)), C.c_double(t),
            _abi.ptr(orank), _abi.ptr(oidx), C.byref(n)))
        return list(zip(orank[: n.value].tolist(), oidx[: n.value].tolist()))

    def close(self):
        if self.h:
            lib().csg_store_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Model tables
# ---------------------------------------------------------------------------
class Model:
    def __init__(self, topo: Topology, prog: OpProgram, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.topo, self.prog = topo, prog
        td, k1 = topo.desc()
        pd, k2 = prog.desc()
        self.h = C.c_void_p()
        _check(lib().csg_model_create(self.ctx.h, C.byref(td), C.byref(pd),
                                      C.byref(self.h)))

    def close(self):
        if self.h:
            lib().csg_model_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_layout(tp, pp, dp, ranks_per_node, channels_per_pair, nics_per_node=4,
                 msg_bytes=64 << 20) -> Tuple[Topology, OpProgram]:
    """build_layout + default_program (host C++ of this build)."""
    js = C.c_void_p()
    _ccheck(lib().collsight_b200_layout_json(tp, pp, dp, ranks_per_node,
                                             channels_per_pair, nics_per_node,
                                             C.c_uint64(msg_bytes), C.byref(js)))
    text = C.string_at(js.value).decode()
    lib().collsight_b200_free(js)
    return layout_from_json(text, tp, pp, dp)


def sample_ranks(model: Model, max_sampled: int, seed: int) -> List[int]:
    out = np.zeros(len(model.topo.groups) + 1, dtype=np.int32)
    n = C.c_size_t()
    _check(lib().csg_sample_ranks(model.h, C.c_int32(max_sampled), C.c_uint64(seed),
                                  _abi.ptr(out), C.c_size_t(len(out)), C.byref(n)))
    return out[: n.value].tolist()


# ---------------------------------------------------------------------------
# Trigger (proj/include/collsight/trigger.hpp)
# ---------------------------------------------------------------------------
class TriggerState:
    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.h = C.c_void_p()
        _check(lib().csg_trigger_state_create(self.ctx.h, C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                lib().csg_trigger_state_free(self.h)
        except Exception:
            pass


def evaluate(store: TraceStore, sampled: Sequence[int], t: float,
             state: TriggerState, cfg: TriggerConfig) -> Optional[TriggerEvent]:
    s = np.ascontiguousarray(sampled, dtype=np.int32)
    tripped = C.c_int()
    ev = _abi.TriggerEventC()
    tc = cfg.c()
    _check(lib().csg_evaluate(store.h, _abi.ptr(s), C.c_size_t(len(s)), C.c_double(t),
                              state.h, C.byref(tc), C.byref(tripped), C.byref(ev)))
    if not tripped.value:
        return None
    return TriggerEvent(ev.kind, ev.suspect_rank, ev.time_ms)


# ---------------------------------------------------------------------------
# Reports
# ---------------------------------------------------------------------------
def _entry(s: _abi.SuspectC) -> dict:
    return {"rank": s.rank, "category": s.category, "side": s.side,
            "group": s.group, "op_seq": s.stuck_op, "onset_ms": s.onset_ms}


def _report(v: _abi.ReportViewC) -> dict:
    """csg_report_view -> the structured report dict (same schema as the
    oracle's full report: RootCauseReport, proj/include/collsight/rca.hpp)."""
    return {
        "verdict": v.verdict,
        "kind": v.trigger.kind,
        "suspect_rank": v.trigger.suspect_rank,
        "time_ms": v.trigger.time_ms,
        "suspects": [_entry(v.suspects[i]) for i in range(v.n_suspects)],
        "exonerated": [_entry(v.exonerated[i]) for i in range(v.n_exonerated)],
        "affected_groups": [v.affected_groups[i] for i in range(v.n_affected)],
        "evidence": [{"rank": v.evidence[i].rank, "channel": v.evidence[i].channel,
                      "time_ms": v.evidence[i].time_ms,
                      "op_seq": v.evidence[i].op_seq} for i in range(v.n_evidence)],
        "records_scanned": v.records_scanned,
    }


def _take_results(h: C.c_void_p) -> List[dict]:
    try:
        n = lib().csg_results_count(h)
        out = []
        for i in range(n):
            v = _abi.ReportViewC()
            _check(lib().csg_results_get(h, C.c_size_t(i), C.byref(v)))
            out.append(_report(v))
        return out
    finally:
        lib().csg_results_free(h)


def analyze(store: TraceStore, model: Model, cfg: AnalysisConfig,
            trigger: TriggerEvent, mode: int = 0) -> dict:
    """analyze (mode 0) / analyze_failure (1) / analyze_straggler (2)."""
    ac = cfg.c()
    tr = trigger.c()
    h = C.c_void_p()
    _check(lib().csg_analyze(store.h, model.h, C.byref(ac), C.byref(tr), C.c_int(mode),
                             C.byref(h)))
    return _take_results(h)[0]


def analyze_failure(store, model, cfg, trigger) -> dict:
    return analyze(store, model, cfg, trigger, 1)


def analyze_straggler(store, model, cfg, trigger) -> dict:
    return analyze(store, model, cfg, trigger, 2)


def affected_groups(store: TraceStore, model: Model, cfg: AnalysisConfig,
                    trigger: TriggerEvent) -> Tuple[List[int], int]:
    ac = cfg.c()
    tr = trigger.c()
    out = np.zeros(max(1, len(model.topo.groups)), dtype=np.int32)
    n = C.c_size_t()
    sc = C.c_uint64(0)
    _check(lib().csg_affected_groups(store.h, model.h, C.byref(ac), C.byref(tr),
                                     _abi.ptr(out), C.c_size_t(len(out)), C.byref(n),
                                     C.byref(sc)))
    return out[: n.value].tolist(), sc.value


class Results:
    """Host-resident csg_results of one detection replay; report dicts are
    built on demand (the replay itself has finished when this exists)."""

    def __init__(self, h: C.c_void_p):
        self._h = h

    def __len__(self) -> int:
        return int(lib().csg_results_count(self._h)) if self._h else 0

    def reports(self) -> List[dict]:
        h, self._h = self._h, None
        return _take_results(h) if h else []

    def jsonl(self, scenario: "Scenario") -> str:
        """reports_to_jsonl bytes under the scenario's config, rendered in C++
        (collsight_b200_results_jsonl); the results stay usable."""
        if not self._h:
            raise EngineError(5, "results already consumed")
        js = C.c_void_p()
        _ccheck(lib().collsight_b200_results_jsonl(scenario.h, self._h, C.byref(js)))
        try:
            return C.string_at(js.value).decode()
        finally:
            lib().collsight_b200_free(js)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().csg_results_free(self._h)
            self._h = None


def run_detection_results(store: TraceStore, model: Model, tcfg: TriggerConfig,
                          acfg: AnalysisConfig, seed: int):
    """-> (Results, sampled ranks); the reports stay in host C structs."""
    tc, ac = tcfg.c(), acfg.c()
    h = C.c_void_p()
    sampled = np.zeros(len(model.topo.groups) + 1, dtype=np.int32)
    ns = C.c_size_t()
    _check(lib().csg_run_detection(store.h, model.h, C.byref(tc), C.byref(ac),
                                   C.c_uint64(seed), C.byref(h), _abi.ptr(sampled),
                                   C.c_size_t(len(sampled)), C.byref(ns)))
    return Results(h), sampled[: ns.value].tolist()


def run_detection(store: TraceStore, model: Model, tcfg: TriggerConfig,
                  acfg: AnalysisConfig, seed: int):
    """-> (list of report dicts, sampled ranks)"""
    res, sampled = run_detection_results(store, model, tcfg, acfg, seed)
    return res.reports(), sampled


def check_min_op(pairs):
    if not pairs:
        r = np.zeros(1, np.int32)
        o = np.zeros(1, np.int64)
    else:
        r = np.array([a for a, _ in pairs], dtype=np.int32)
        o = np.array([b for _, b in pairs], dtype=np.int64)
    out = np.zeros(max(1, len(pairs)), dtype=np.int32)
    n = C.c_size_t()
    has = C.c_int()
    _check(lib().csg_check_min_op(_abi.ptr(r), _abi.ptr(o), C.c_size_t(len(pairs)),
                                  _abi.ptr(out), C.byref(n), C.byref(has)))
    return out[: n.value].tolist() if has.value else None


def check_min_data(pairs):
    r = np.array([a for a, _ in pairs] or [0], dtype=np.int32)
    pr = (_abi.ProgressC * max(1, len(pairs)))()
    for i, (_, t) in enumerate(pairs):
        pr[i] = _abi.ProgressC(*t)
    out = np.zeros(max(1, len(pairs)), dtype=np.int32)
    n = C.c_size_t()
    _check(lib().csg_check_min_data(_abi.ptr(r), pr, C.c_size_t(len(pairs)),
                                    _abi.ptr(out), C.byref(n)))
    return out[: n.value].tolist()


def check_rc_table(c, peer=None):
    a = _abi.ProgressC(*c)
    b = _abi.ProgressC(*peer) if peer is not None else None
    cat = C.c_int()
    side = C.c_int()
    _check(lib().csg_check_rc_table(C.byref(a), C.byref(b) if b is not None else None,
                                    C.byref(cat), C.byref(side)))
    return cat.value, side.value


# ---------------------------------------------------------------------------
# C API (collsight.h) — scenario-driven runs
# ---------------------------------------------------------------------------
@dataclass
class RunResult:
    text: str
    summary_json: str
    reports_jsonl: str
    trigger_count: int


class Scenario:
    def __init__(self, h: C.c_void_p):
        self.h = h

    @classmethod
    def load(cls, path: str) -> "Scenario":
        h = C.c_void_p()
        _ccheck(lib().collsight_scenario_load(path.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def parse(cls, text: str) -> "Scenario":
        h = C.c_void_p()
        _ccheck(lib().collsight_scenario_parse(text.encode(), C.byref(h)))
        return cls(h)

    def set_seed(self, seed: int):
        _ccheck(lib().collsight_scenario_set_seed(self.h, C.c_uint64(seed)))

    def layout(self) -> Tuple[Topology, OpProgram]:
        js = C.c_void_p()
        _ccheck(lib().collsight_b200_scenario_layout_json(self.h, C.byref(js)))
        text = C.string_at(js.value).decode()
        lib().collsight_b200_free(js)
        return layout_from_json(text)

    def configs(self) -> Tuple[TriggerConfig, AnalysisConfig, int]:
        tc = _abi.TriggerConfigC()
        ac = _abi.AnalysisConfigC()
        seed = C.c_uint64()
        _ccheck(lib().collsight_b200_scenario_configs(self.h, C.byref(tc), C.byref(ac),
                                                      C.byref(seed)))
        t = TriggerConfig(tc.delta_ms, tc.detect_interval_ms, tc.throughput_drop_factor,
                          tc.interval_inflation_factor, tc.max_sampled_ranks,
                          tc.ema_alpha, tc.warmup_windows)
        a = AnalysisConfig(ac.straggler_threshold_ms, ac.consecutive_iterations_k,
                           ac.delta_ms, ac.flow_skew_factor)
        return t, a, seed.value

    def __del__(self):
        try:
            if self.h:
                lib().collsight_scenario_free(self.h)
        except Exception:
            pass


def _take_run(h: C.c_void_p) -> RunResult:
    L = lib()
    try:
        return RunResult(L.collsight_result_text(h).decode(),
                         L.collsight_result_summary_json(h).decode(),
                         L.collsight_result_reports_jsonl(h).decode(),
                         L.collsight_result_trigger_count(h))
    finally:
        L.collsight_result_free(h)


def run_analyze(scenario: Scenario, trace_path: str,
                report_path: Optional[str] = None) -> RunResult:
    h = C.c_void_p()
    _ccheck(lib().collsight_run_analyze(scenario.h, trace_path.encode(),
                                        report_path.encode() if report_path else None,
                                        C.byref(h)))
    return _take_run(h)


def run_analyze_packed(scenario: Scenario, records: np.ndarray,
                       report_path: Optional[str] = None) -> RunResult:
    r = np.ascontiguousarray(records, dtype=_abi.RECORD_DTYPE)
    h = C.c_void_p()
    _ccheck(lib().collsight_b200_run_analyze_packed(
        scenario.h, _abi.ptr(r), C.c_size_t(len(r)),
        report_path.encode() if report_path else None, C.byref(h)))
    return _take_run(h)


def jsonl_parse_line(line) -> Optional[np.ndarray]:
    """Host instantiation of the device line parser: the record, or None
    when it defers to the exact parser."""
    b = line.encode() if isinstance(line, str) else bytes(line)
    out = np.zeros(1, dtype=_abi.RECORD_DTYPE)
    ok = lib().csg_jsonl_parse_line(b, C.c_size_t(len(b)), _abi.ptr(out))
    return out if ok else None


def jsonl_parse_double(tok) -> Optional[float]:
    b = tok.encode() if isinstance(tok, str) else bytes(tok)
    d = C.c_double()
    ok = lib().csg_jsonl_parse_double(b, C.c_size_t(len(b)), C.byref(d))
    return d.value if ok else None


def serialize_records(records: np.ndarray, ranks_per_node: int = 8) -> str:
    """Packed records -> reference-format JSONL (collsight_b200_serialize_trace)."""
    r = np.ascontiguousarray(records, dtype=_abi.RECORD_DTYPE)
    out = C.c_void_p()
    n = C.c_size_t()
    _ccheck(lib().collsight_b200_serialize_trace(_abi.ptr(r), C.c_size_t(len(r)),
                                                 C.c_int32(ranks_per_node), C.byref(out),
                                                 C.byref(n)))
    try:
        return C.string_at(out.value, n.value).decode()
    finally:
        lib().collsight_b200_free(out)


def write_trace(records: np.ndarray, path: str, ranks_per_node: int = 8) -> None:
    """Packed records -> a reference-format JSONL trace file."""
    r = np.ascontiguousarray(records, dtype=_abi.RECORD_DTYPE)
    _ccheck(lib().collsight_b200_write_trace(_abi.ptr(r), C.c_size_t(len(r)),
                                             C.c_int32(ranks_per_node), path.encode()))


def parse_trace(text: str) -> np.ndarray:
    b = text.encode()
    out = C.c_void_p()
    n = C.c_size_t()
    _ccheck(lib().collsight_b200_parse_trace(b, C.c_size_t(len(b)), C.byref(out),
                                             C.byref(n)))
    try:
        return np.frombuffer(C.string_at(out.value, n.value * 48),
                             dtype=_abi.RECORD_DTYPE).copy()
    finally:
        lib().collsight_b200_free(out)


def synthesize(scenario: Scenario, target_records: int = 0,
               rank_range: Optional[Tuple[int, int]] = None) -> np.ndarray:
    """Synthetic trace for the scenario (benchmark generator, synth.cpp);
    rank_range=(lo, hi) keeps one shard's records."""
    out = C.c_void_p()
    n = C.c_size_t()
    lo, hi = rank_range if rank_range else (0, 0x7FFFFFFF)
    _ccheck(lib().collsight_b200_synthesize_ranks(scenario.h, C.c_uint64(target_records),
                                                  C.c_int32(lo), C.c_int32(hi),
                                                  C.byref(out), C.byref(n)))
    try:
        arr = np.empty(n.value, dtype=_abi.RECORD_DTYPE)
        if n.value:
            C.memmove(arr.ctypes.data, out.value, n.value * 48)
        return arr
    finally:
        lib().collsight_b200_free(out)


def synthesize_into(store: "TraceStore", scenario: Scenario, target_records: int = 0,
                    rank_range: Optional[Tuple[int, int]] = None) -> int:
    """The same synthetic records as synthesize(), generated on the store's
    GPU (synth_gpu.cu) and appended to the store; returns how many."""
    n = C.c_uint64()
    lo, hi = rank_range if rank_range else (0, 0x7FFFFFFF)
    _ccheck(lib().collsight_b200_synthesize_store(scenario.h, C.c_uint64(target_records),
                                                  C.c_int32(lo), C.c_int32(hi), store.h,
                                                  C.byref(n)))
    return n.value


def comm_unique_id() -> bytes:
    """NCCL unique id for csg_ctx_comm_init (call on one rank, broadcast)."""
    buf = (C.c_ubyte * 128)()
    _check(lib().csg_comm_unique_id(buf, C.c_size_t(128)))
    return bytes(buf)
