"""Host-side layout / program / config mirrors.

Python mirrors of the reference types the analyzer API takes:
Topology + CommGroup (reference proj/include/collsight/topology.hpp:15-55),
OpProgram + CollOpSpec (proj/include/collsight/program.hpp:14-30),
TriggerConfig (trigger.hpp:15-25), AnalysisConfig (rca.hpp:42-49) and
TriggerEvent (trigger.hpp:39-43). They lower to the plain-C descriptors of
include/csg_engine.h; no analysis happens here.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi


@dataclass
class CommGroup:
    comm_id: int
    kind: int  # 0 DP, 1 PP, 2 TP
    members: List[int]


@dataclass
class Topology:
    world_size: int
    groups: List[CommGroup]
    tp: int = 0
    pp: int = 0
    dp: int = 0

    def groups_of(self, rank: int) -> List[int]:
        return [g.comm_id for g in self.groups if rank in g.members]

    def group_of(self, rank: int, kind: int) -> CommGroup:
        for g in self.groups:
            if g.kind == kind and rank in g.members:
                return g
        raise KeyError(rank)

    def desc(self):
        """-> (TopologyDesc, keep-alive arrays)."""
        kinds = np.array([g.kind for g in self.groups], dtype=np.uint8)
        off = np.zeros(len(self.groups) + 1, dtype=np.int64)
        for i, g in enumerate(self.groups):
            off[i + 1] = off[i] + len(g.members)
        mem = np.array([m for g in self.groups for m in g.members], dtype=np.int32)
        d = _abi.TopologyDesc(self.world_size, len(self.groups), _abi.ptr(kinds),
                              _abi.ptr(off), _abi.ptr(mem))
        return d, (kinds, off, mem)


@dataclass
class CollOpSpec:
    op_seq: int
    op_name: int
    group: int
    depends_on: List[int] = field(default_factory=list)
    src: int = -1
    dst: int = -1


@dataclass
class OpProgram:
    ops: List[CollOpSpec]

    def ops_per_iteration(self) -> int:
        return len(self.ops)

    def desc(self):
        n = len(self.ops)
        names = np.array([o.op_name for o in self.ops], dtype=np.uint8)
        grp = np.array([o.group for o in self.ops], dtype=np.int32)
        src = np.array([o.src for o in self.ops], dtype=np.int32)
        dst = np.array([o.dst for o in self.ops], dtype=np.int32)
        off = np.zeros(n + 1, dtype=np.int64)
        for i, o in enumerate(self.ops):
            off[i + 1] = off[i] + len(o.depends_on)
        deps = np.array([d for o in self.ops for d in o.depends_on], dtype=np.int64)
        d = _abi.ProgramDesc(n, _abi.ptr(names), _abi.ptr(grp), _abi.ptr(src),
                             _abi.ptr(dst), _abi.ptr(off), _abi.ptr(deps))
        return d, (names, grp, src, dst, off, deps)


@dataclass
class TriggerConfig:
    delta_ms: float = 200.0
    detect_interval_ms: float = 500.0
    throughput_drop_factor: float = 0.5
    interval_inflation_factor: float = 2.0
    max_sampled_ranks: int = 10
    ema_alpha: float = 0.3
    warmup_windows: int = 3

    def c(self) -> _abi.TriggerConfigC:
        return _abi.TriggerConfigC(self.delta_ms, self.detect_interval_ms,
                                   self.throughput_drop_factor,
                                   self.interval_inflation_factor,
                                   self.max_sampled_ranks, self.warmup_windows,
                                   self.ema_alpha)


@dataclass
class AnalysisConfig:
    straggler_threshold_ms: float = 1000.0
    consecutive_iterations_k: int = 3
    delta_ms: float = 200.0
    flow_skew_factor: float = 2.0

    def c(self) -> _abi.AnalysisConfigC:
        return _abi.AnalysisConfigC(self.straggler_threshold_ms, self.delta_ms,
                                    self.flow_skew_factor,
                                    self.consecutive_iterations_k, 0)


FAILURE, STRAGGLER = 0, 1


@dataclass
class TriggerEvent:
    kind: int
    suspect_rank: int
    time_ms: float

    def c(self) -> _abi.TriggerEventC:
        return _abi.TriggerEventC(self.kind, self.suspect_rank, self.time_ms)


def layout_from_json(text: str, tp=0, pp=0, dp=0):
    """Parse the {"world_size", "groups", "ops"} layout JSON emitted by the
    host library (and by the oracle shim) into Topology + OpProgram."""
    j = json.loads(text)
    topo = Topology(j["world_size"],
                    [CommGroup(i, g["kind"], list(g["members"]))
                     for i, g in enumerate(j["groups"])], tp, pp, dp)
    prog = OpProgram([CollOpSpec(i, o["name"], o["group"], list(o["deps"]),
                                 o["src"], o["dst"])
                      for i, o in enumerate(j["ops"])])
    return topo, prog


# ---------------------------------------------------------------------------
# Record builders (the test helpers of proj/tests/test_rca.cpp:15-51 and
# test_trigger.cpp:14-46 take the same arguments).
# ---------------------------------------------------------------------------
def records(n: int = 0) -> np.ndarray:
    return np.zeros(n, dtype=_abi.RECORD_DTYPE)


def completion(rank, comm_id, op_seq, start_ms, end_ms, channel=0,
               msg_bytes=1 << 20, op_name=_abi.OP_ALLGATHER) -> np.ndarray:
    r = records(1)
    r["ts"] = end_ms
    r["op_seq"] = op_seq
    r["rank"] = rank
    r["comm_id"] = comm_id
    r["channel"] = channel
    r["kind"] = _abi.KIND_COMPLETION
    r["op_name"] = op_name
    r["start_ms"] = start_ms
    r["msg_bytes"] = msg_bytes
    return r


def state(rank, comm_id, op_seq, window_end_ms, staged, transmitted, done,
          channel=0) -> np.ndarray:
    r = records(1)
    r["ts"] = window_end_ms
    r["op_seq"] = op_seq
    r["rank"] = rank
    r["comm_id"] = comm_id
    r["channel"] = channel
    r["kind"] = _abi.KIND_STATE
    r["gpu_ready"] = staged
    r["rdma_transmitted"] = transmitted
    r["rdma_done"] = done
    return r


def concat(*recs) -> np.ndarray:
    if not recs:
        return records(0)
    return np.concatenate([np.atleast_1d(r) for r in recs]).astype(_abi.RECORD_DTYPE)
