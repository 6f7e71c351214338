"""Hand-built layouts and record builders mirroring the reference's unit-test
fixtures (proj/tests/test_rca.cpp:15-98, :298-381; test_trigger.cpp:14-63;
test_trace.cpp:15-66)."""
from __future__ import annotations

import numpy as np

from paper_2509_03018_b200 import _abi
from paper_2509_03018_b200.model import (AnalysisConfig, CollOpSpec, CommGroup,
                                         OpProgram, Topology, completion, concat,
                                         records, state)

AG, RS, AR, SEND, RECV = range(5)


def fig5():
    """GPUs 1,2,3 form a DP group; GPUs 2,4 a PP group (test_rca.cpp:55-98)."""
    topo = Topology(5, [CommGroup(0, 0, [1, 2, 3]), CommGroup(1, 1, [2, 4])])
    prog = OpProgram([CollOpSpec(0, AG, 0),
                      CollOpSpec(1, SEND, 1, [0], 2, 4),
                      CollOpSpec(2, RECV, 1, [1], 2, 4)])
    return topo, prog, AnalysisConfig(delta_ms=500)


def fig5_slow_gpu1():
    recs = []
    for r in (1, 2, 3):
        recs.append(completion(r, 0, 0, 400, 450))
    recs.append(completion(2, 1, 1, 455, 470))
    recs.append(completion(4, 1, 2, 455, 470))
    for w in (600.0, 800.0):
        v = 2 if w > 700 else 1
        recs.append(state(1, 0, 3, w, v, v, v))
        recs.append(state(2, 0, 3, w, 5, 5, 5))
        recs.append(state(3, 0, 3, w, 5, 5, 5))
        recs.append(state(4, 1, 5, w, 0, 0, 0))
    return concat(*recs)


def two_group():
    """Group A {0,1} feeds group B {2,3} (test_rca.cpp:298-342)."""
    topo = Topology(4, [CommGroup(0, 0, [0, 1]), CommGroup(1, 0, [2, 3])])
    prog = OpProgram([CollOpSpec(0, AG, 0), CollOpSpec(1, AG, 1, [0])])
    recs = concat(state(0, 0, 0, 600, 1, 1, 1), state(1, 0, 0, 600, 3, 3, 3),
                  state(2, 1, 1, 650, 0, 0, 0), state(3, 1, 1, 650, 0, 0, 0))
    return topo, prog, AnalysisConfig(delta_ms=500), recs


class Straggler:
    """3-rank TP group, one AllGather per iteration (test_rca.cpp:348-381)."""

    def __init__(self):
        self.topo = Topology(3, [CommGroup(0, 2, [0, 1, 2])])
        self.prog = OpProgram([CollOpSpec(0, AG, 0)])
        self.cfg = AnalysisConfig(delta_ms=100000)
        self.recs = []

    def add_iteration(self, j, off0, off1, off2, shift=0.0):
        base = shift + 10000.0 * j
        self.recs.append(completion(0, 0, j, base + off0, base + off0 + 100))
        self.recs.append(completion(1, 0, j, base + off1, base + off1 + 100))
        self.recs.append(completion(2, 0, j, base + off2, base + off2 + 100))

    def store(self):
        return concat(*self.recs)


def trig_completion(rank, end, nbytes, op=0):
    """test_trigger.cpp:14-30"""
    r = completion(rank, 0, op, end - 1 if end > 1 else 0, end, 0, int(nbytes))
    return r


def trig_state(rank, window_end, op=1):
    """test_trigger.cpp:32-46"""
    return state(rank, 0, op, window_end, 4, 4, 4)


def random_records(rng: np.random.Generator, n: int, ranks=32, tmax=20000.0,
                   ops=64, channels=4, comms=4) -> np.ndarray:
    """Random store in the spirit of test_trace.cpp:52-66 (values valid per
    validate_record, timestamps on a coarse grid so ties occur)."""
    r = records(n)
    kind = rng.integers(0, 2, n)
    r["kind"] = kind
    r["rank"] = rng.integers(0, ranks, n)
    r["comm_id"] = rng.integers(0, comms, n)
    r["channel"] = rng.integers(0, channels, n)
    r["op_seq"] = rng.integers(0, ops, n)
    ts = np.round(rng.uniform(0, tmax, n) / 2.5) * 2.5
    r["ts"] = ts
    comp = kind == 0
    start = ts - np.round(rng.uniform(0, 50, n), 1)
    r["op_name"] = np.where(comp, rng.integers(0, 5, n), 0)
    st = np.where(comp, start, 0.0)
    mb = np.where(comp, rng.integers(1, 1 << 24, n), 0).astype(np.uint64)
    ready = rng.integers(0, 9, n)
    tx = (ready * rng.uniform(0, 1, n)).astype(np.int64)
    done = (tx * rng.uniform(0, 1, n)).astype(np.int64)
    # union payload: write completion fields, then overwrite states' lanes
    r["start_ms"] = st
    r["msg_bytes"] = mb
    s = ~comp
    raw = r.view(np.uint8).reshape(-1, 48)
    lanes = np.zeros((n, 4), dtype=np.uint32)
    lanes[:, 0] = ready
    lanes[:, 1] = tx
    lanes[:, 2] = done
    raw[s, 32:48] = lanes[s].view(np.uint8).reshape(-1, 16)
    return r
