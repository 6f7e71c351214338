"""Pins the CPU restatement (oracle/restate.py) to the reference: it must
reproduce the reference's structured reports on the catalog fixtures and the
known-answer stores, and agree with the compiled reference (oracle/_ref) on
queries and trigger sequences. CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import restate as RS
from paper_2509_03018_b200.model import (AnalysisConfig, TriggerConfig, TriggerEvent,
                                         concat, completion, state)
from tests import fixtures as fx
from tests.conftest import GOLDEN
from tests.golden import codec

LAYOUT = dict(tp=8, pp=2, dp=2, rpn=8, cpp=2, nics=4)


def _catalog_model(oracle):
    topo, prog = oracle.layout(8, 2, 2, 8, 2, 4, 67108864)
    return topo, prog, RS.model_from(topo, prog)


def _configs(name):
    cfg = json.load(open(os.path.join(GOLDEN, "configs", name + ".json")))
    tr = cfg.get("trigger", {})
    d = tr.get("delta_ms", 2 * cfg["sim"]["state_log_window_ms"])
    tcfg = TriggerConfig(delta_ms=d, detect_interval_ms=tr.get("detect_interval_ms", 500.0),
                         max_sampled_ranks=tr.get("max_sampled_ranks", 10))
    an = cfg.get("analysis", {})
    acfg = AnalysisConfig(delta_ms=an.get("delta_ms", d),
                          straggler_threshold_ms=an.get("straggler_threshold_ms", 1000.0))
    return tcfg, acfg, cfg["seed"]


@pytest.mark.parametrize("name", ["clean", "scenario1", "scenario3", "scenario5",
                                  "scenario7"])
def test_restatement_reproduces_reference_catalog(oracle, name):
    recs = codec.load_file(os.path.join(GOLDEN, f"catalog_{name}.rec.xz"))
    full = [json.loads(l) for l in open(os.path.join(GOLDEN, f"catalog_{name}.full.jsonl"))]
    topo, prog, m = _catalog_model(oracle)
    tcfg, acfg, seed = _configs(name)
    got, sampled = RS.run_detection(recs, m, tcfg, acfg, seed)
    assert sampled == json.load(open(os.path.join(GOLDEN, "manifest.json")))[name]["sampled"]
    assert got == full


def test_restatement_kats(oracle):
    topo, prog, cfg = fx.fig5()
    m = RS.model_from(topo, prog)
    recs = fx.fig5_slow_gpu1()
    st = RS.Store(recs)
    assert RS.affected_groups(st, m, cfg, (0, 4, 800.0)) == [0, 1]
    assert RS.analyze_failure(st, m, cfg, (0, 4, 800.0)) == \
        oracle.analyze(topo, prog, cfg, recs, TriggerEvent(0, 4, 800.0), 1)
    topo, prog, cfg, recs = fx.two_group()
    assert RS.analyze_failure(RS.Store(recs), RS.model_from(topo, prog), cfg, (0, 2, 900.0)) \
        == oracle.analyze(topo, prog, cfg, recs, TriggerEvent(0, 2, 900.0), 1)
    fix = fx.Straggler()
    for j in range(4):
        fix.add_iteration(j, 0, 50, 1250)
    recs = fix.store()
    assert RS.analyze_straggler(RS.Store(recs), RS.model_from(fix.topo, fix.prog), fix.cfg,
                                (1, 0, 40000.0)) == \
        oracle.analyze(fix.topo, fix.prog, fix.cfg, recs, TriggerEvent(1, 0, 40000.0), 2)


def test_restatement_table_functions(oracle):
    for c in [(0, 0, 0), (5, 3, 3), (5, 5, 5), (5, 5, 3), (4, 2, 1)]:
        for peer in [None, (5, 5, 5), (3, 3, 1)]:
            assert RS.check_rc_table(c, peer) == oracle.check_rc_table(c, peer)
    assert RS.check_min_op([(0, 42), (1, 41), (2, 42)]) == [1]
    assert RS.check_min_op([(0, 4), (1, 4)]) is None


def test_restatement_query_and_trigger(oracle):
    rng = np.random.default_rng(101)
    recs = fx.random_records(rng, 1000, tmax=10000.0)
    st = RS.Store(recs)
    for _ in range(30):
        t0 = float(rng.integers(0, 10000))
        t1 = t0 + float(rng.integers(0, 4000))
        ranks = [r for r in range(32) if rng.integers(0, 3) == 0] or [0]
        assert RS.query(st, ranks, t0, t1) == oracle.query(recs, ranks, t0, t1)
        tt = float(rng.integers(0, 20000))
        assert RS.last_log_per_rank(st, list(range(32)), tt) == \
            oracle.last_log_per_rank(recs, list(range(32)), tt)
    cfg = TriggerConfig(delta_ms=300.0, warmup_windows=2)
    s1, s2 = RS.TriggerState(), oracle.TriggerState()
    for k in range(1, 34):
        got = RS.evaluate(st, [1, 4, 9, 17], 300.0 * k, s1, cfg)
        want = oracle.evaluate(recs, [1, 4, 9, 17], 300.0 * k, s2, cfg)
        assert (got is None) == (want is None)
        if got:
            assert got == (want.kind, want.suspect_rank, want.time_ms)
