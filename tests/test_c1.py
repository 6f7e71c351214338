"""C1 parity: the 32-rank ring AllReduce trace, 4 channels,
1000 one-op iterations, one injected slow NIC — plus a factor-0.01 variant
and a NIC-shutdown hang on the same ring (tests/golden/make_c1.py).

The golden traces and reports come from the reference simulator and the
reference run_detection over the custom AllReduce program (proj/src/
runner.cpp:47-81). The CPU test pins the fixtures to the reference itself
(oracle/_ref) — the trace is regenerated and both hashes must match — and the
GPU test requires the B200 engine to reproduce the structured reports
(suspects, exonerated, affected groups, evidence, records_scanned) exactly.
"""
import json
import os

import pytest

from tests.conftest import GOLDEN
from tests.golden import codec

VARIANTS = ["c1_ring_32", "c1_ring_32_f001", "c1_ring_32_hang"]
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


def golden(name):
    recs = codec.load_file(os.path.join(GOLDEN, f"{name}.rec.xz"))
    full = [json.loads(l) for l in open(os.path.join(GOLDEN, f"{name}.full.jsonl"))]
    return recs, full


def layout():
    """The reference build_layout(1, 1, 32, 1, 4, 4) tables, as the engine's
    scenario layout renders them; the program is the custom one-op AllReduce."""
    from paper_2509_03018_b200 import engine
    from tests.golden.make_c1 import program
    scen = engine.Scenario.load(os.path.join(GOLDEN, "configs", "c1_ring_32.json"))
    topo, _ = scen.layout()
    return topo, program(), scen


def test_c1_layout_is_one_ring():
    topo, prog, _ = layout()
    assert topo.world_size == 32
    assert len(topo.groups) == 65
    assert topo.groups[0].members == list(range(32))
    assert all(len(g.members) == 1 for g in topo.groups[1:])
    assert prog.ops_per_iteration() == 1


@pytest.mark.parametrize("name", VARIANTS)
def test_c1_fixture_pinned_to_reference(oracle, name):
    from tests.golden.make_c1 import MSG_BYTES, config_text, program
    from tests.golden.make_golden import fnv1a64
    recs = oracle.simulate_prog(config_text(name), program(), MSG_BYTES)
    assert fnv1a64(recs.tobytes()) == MANIFEST[name]["records_fnv1a64"]
    want, _ = golden(name)
    assert (recs == want).all()


def test_c1_reports_pinned_to_reference(oracle):
    """Reference run_detection over the committed trace reproduces the
    committed reports (one variant per CPU run keeps the suite short)."""
    from tests.golden.make_golden import fnv1a64
    name = "c1_ring_32"
    recs, full = golden(name)
    topo, prog, scen = layout()
    tcfg, acfg, seed = scen.configs()
    reports, got, _ = oracle.run_detection(topo, prog, tcfg, acfg, seed, recs,
                                           onset=30004.0)
    assert got == full
    assert fnv1a64(reports.encode()) == MANIFEST[name]["reports_fnv1a64"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", VARIANTS)
def test_c1_structured_reports(eng, name):
    recs, full = golden(name)
    assert len(recs) == MANIFEST[name]["records"]
    topo, prog, _ = layout()
    cfg = json.loads(open(os.path.join(GOLDEN, "configs", name + ".json")).read())
    tcfg, acfg, seed = eng.Scenario.parse(json.dumps(cfg)).configs()
    store = eng.TraceStore(records=recs)
    model = eng.Model(topo, prog)
    got, sampled = eng.run_detection(store, model, tcfg, acfg, seed)
    assert len(got) == len(full)
    for i, (a, b) in enumerate(zip(got, full)):
        assert a == b, (i, a, b)
