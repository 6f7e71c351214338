"""GPU ports of the reference's known-answer unit tests
(proj/tests/test_trace.cpp, test_trigger.cpp, test_rca.cpp), run through the
engine's C ABI. Where the oracle library is present each case is also
compared field by field against the reference's own output."""
import numpy as np
import pytest

from paper_2509_03018_b200.model import (FAILURE, STRAGGLER, AnalysisConfig,
                                         CommGroup, TriggerConfig, TriggerEvent,
                                         completion, concat, state)
from tests import fixtures as fx

GPU_ISSUE, LATE_START, FLOW_SKEWED = 3, 4, 7
V_SUSPECTS, V_UNDET, V_FALSE, V_INSUFF, V_NOSTRAG = range(5)

pytestmark = pytest.mark.gpu


def oracle_or_none():
    from oracle import ref
    return ref if ref.available() else None


# ---------------------------------------------------------------- trace ----

def test_query_matches_brute_force(eng):
    rng = np.random.default_rng(3)
    recs = fx.random_records(rng, 1000, tmax=10000.0)
    store = eng.TraceStore(records=recs)
    ts, rk = recs["ts"], recs["rank"]
    ref = oracle_or_none()
    for _ in range(100):
        t0 = float(rng.integers(0, 10000))
        t1 = t0 + float(rng.integers(0, 4000))
        ranks = [r for r in range(32) if rng.integers(0, 3) == 0] or [0]
        idx = [i for i in range(len(recs)) if t0 <= ts[i] <= t1 and rk[i] in ranks]
        idx.sort(key=lambda i: (ts[i], rk[i]))  # stable on store order
        got = store.query(ranks, t0, t1)
        assert got == idx
        if ref:
            assert got == ref.query(recs, ranks, t0, t1)
    with pytest.raises(eng.EngineError) as e:
        store.query([0], 10.0, 5.0)
    assert e.value.status == 4 and e.value.msg == "query: t0 > t1"


def test_query_on_empty_store(eng):
    assert eng.TraceStore().query([0, 1], 0.0, 100.0) == []


def test_last_log_per_rank(eng):
    recs = [completion(0, 1, 5, 9.0, 10.0), state(0, 1, 6, 11.0, 1, 1, 1),
            completion(1, 1, 9, 49.0, 50.0), state(2, 1, 4, 9.0, 1, 1, 1),
            state(2, 1, 5, 9.0, 1, 1, 1)]
    store = eng.TraceStore(records=concat(*recs))
    all_ = concat(*recs)
    last = store.last_log_per_rank([0, 1, 2], 20.0)
    assert [r for r, _ in last] == [0, 2]
    assert [int(all_["op_seq"][i]) for _, i in last] == [6, 5]
    more = recs + [completion(1, 1, 1, 18.0, 19.0), completion(1, 1, 2, 19.0, 20.0)]
    store = eng.TraceStore(records=concat(*more))
    all_ = concat(*more)
    last = store.last_log_per_rank([0, 1, 2], 20.0)
    assert len(last) == 3 and int(all_["op_seq"][last[1][1]]) == 2
    with pytest.raises(eng.EngineError) as e:
        store.last_log_per_rank([], 1.0)
    assert e.value.msg == "last_log_per_rank: empty group"


def test_last_log_matches_brute_force(eng):
    rng = np.random.default_rng(17)
    recs = fx.random_records(rng, 1000)
    store = eng.TraceStore(records=recs)
    ref = oracle_or_none()
    for t in (0.0, 123.4, 5000.0, 20000.0):
        got = store.last_log_per_rank(list(range(32)), t)
        want = []
        for r in range(32):
            best = None
            for i in range(len(recs)):
                if recs["rank"][i] != r or recs["ts"][i] > t:
                    continue
                if best is None or recs["ts"][i] >= recs["ts"][best]:
                    best = i
            if best is not None:
                want.append((r, best))
        assert got == want
        if ref:
            assert got == ref.last_log_per_rank(recs, list(range(32)), t)


# -------------------------------------------------------------- trigger ----

def warm_baseline(eng, recs, st, cfg, rank, bytes_per_window, upto, windows):
    """test_trigger.cpp:50-63"""
    for w in range(windows):
        t = upto - (windows - w) * cfg.delta_ms
        recs.append(fx.trig_completion(rank, t - cfg.delta_ms * 0.75,
                                       bytes_per_window / 2, w * 2))
        recs.append(fx.trig_completion(rank, t - cfg.delta_ms * 0.25,
                                       bytes_per_window / 2, w * 2 + 1))
        store = eng.TraceStore(records=concat(*recs))
        assert eng.evaluate(store, [rank], t, st, cfg) is None


def test_stall_raises_failure(eng):
    cfg = TriggerConfig(delta_ms=100)
    store = eng.TraceStore(records=concat(fx.trig_state(3, 950), fx.trig_state(3, 1000)))
    trig = eng.evaluate(store, [3], 1000, eng.TriggerState(), cfg)
    assert trig == TriggerEvent(FAILURE, 3, 1000.0)


def test_silence_after_activity(eng):
    cfg = TriggerConfig(delta_ms=100)
    st = eng.TriggerState()
    store = eng.TraceStore(records=fx.trig_state(3, 380))
    assert eng.evaluate(store, [3], 400, st, cfg) is not None
    trig = eng.evaluate(store, [3], 500, st, cfg)
    assert trig is not None and trig.kind == FAILURE


def test_cold_start_quiet(eng):
    cfg = TriggerConfig(delta_ms=100)
    assert eng.evaluate(eng.TraceStore(), [0, 1], 200, eng.TriggerState(), cfg) is None


@pytest.mark.parametrize("nbytes,trips", [(5000, True), (5100, False)])
def test_throughput_boundary(eng, nbytes, trips):
    cfg = TriggerConfig(delta_ms=100, warmup_windows=3)
    st = eng.TriggerState()
    recs = []
    warm_baseline(eng, recs, st, cfg, 0, 10000.0, 1000, 4)
    recs.append(fx.trig_completion(0, 1050, nbytes, 100))
    trig = eng.evaluate(eng.TraceStore(records=concat(*recs)), [0], 1100, st, cfg)
    assert (trig is not None) == trips
    if trips:
        assert trig.kind == STRAGGLER


def test_interval_doubling(eng):
    cfg = TriggerConfig(delta_ms=1000, warmup_windows=3)
    st = eng.TriggerState()
    recs = []
    for w in range(4):
        t = 1000.0 * (w + 1)
        for i in range(5):
            recs.append(fx.trig_completion(0, t - 900 + i * 200.0, 20000, w * 10 + i))
        assert eng.evaluate(eng.TraceStore(records=concat(*recs)), [0], t, st, cfg) is None
    for i in range(3):
        recs.append(fx.trig_completion(0, 4200 + i * 400.0, 34000, 100 + i))
    trig = eng.evaluate(eng.TraceStore(records=concat(*recs)), [0], 5000, st, cfg)
    assert trig is not None and trig.kind == STRAGGLER


def test_monotone_threshold(eng):
    cfg = TriggerConfig(delta_ms=100)
    tripped_above = False
    for nbytes in (5200.0, 5100.0, 5000.0, 2500.0, 100.0):
        st = eng.TriggerState()
        recs = []
        warm_baseline(eng, recs, st, cfg, 0, 10000.0, 1000, 4)
        recs.append(fx.trig_completion(0, 1050, nbytes, 100))
        tripped = eng.evaluate(eng.TraceStore(records=concat(*recs)), [0], 1100, st,
                               cfg) is not None
        if not tripped:
            assert not tripped_above
        else:
            tripped_above = True
    assert tripped_above


def test_lowest_rank_wins(eng):
    cfg = TriggerConfig(delta_ms=100)
    store = eng.TraceStore(records=concat(fx.trig_state(5, 1000), fx.trig_state(2, 1000)))
    trig = eng.evaluate(store, [2, 5], 1000, eng.TriggerState(), cfg)
    assert trig.suspect_rank == 2


def test_evaluate_sequences_match_oracle(eng, oracle):
    """Random stores, random sampled lists (duplicates allowed), 40 ticks."""
    rng = np.random.default_rng(29)
    for trial in range(6):
        recs = fx.random_records(rng, 600, ranks=8, tmax=4000.0)
        cfg = TriggerConfig(delta_ms=float(rng.choice([100.0, 300.0])),
                            warmup_windows=int(rng.integers(1, 4)))
        sampled = sorted(rng.integers(0, 10, 4).tolist())
        st_g, st_r = eng.TriggerState(), oracle.TriggerState()
        store = eng.TraceStore(records=recs)
        for k in range(1, 41):
            t = 100.0 * k
            assert eng.evaluate(store, sampled, t, st_g, cfg) == \
                oracle.evaluate(recs, sampled, t, st_r, cfg)


def test_sampling_matches_reference(eng, oracle):
    for shape, seed, cap in [((2, 1, 2, 2, 1, 4), 1, 10), ((8, 2, 2, 8, 2, 4), 7, 10),
                             ((1, 1, 1, 1, 1, 1), 3, 10), ((8, 4, 32, 8, 4, 4), 42, 16),
                             ((8, 2, 2, 8, 2, 4), 11, 3), ((4, 2, 16, 4, 2, 4), 5, 40)]:
        topo, prog = eng.build_layout(*shape)
        m = eng.Model(topo, prog)
        assert eng.sample_ranks(m, cap, seed) == oracle.sample_ranks(topo, cap, seed)


# ------------------------------------------------------------------ rca ----

def test_fig5_affected_and_failure(eng):
    topo, prog, cfg = fx.fig5()
    recs = fx.fig5_slow_gpu1()
    store, model = eng.TraceStore(records=recs), eng.Model(topo, prog)
    trig = TriggerEvent(FAILURE, 4, 800.0)
    groups, scanned = eng.affected_groups(store, model, cfg, trig)
    assert groups == [0, 1] and scanned == len(recs)
    rep = eng.analyze_failure(store, model, cfg, trig)
    assert rep["verdict"] == V_SUSPECTS
    assert [s["rank"] for s in rep["suspects"]] == [1]
    assert rep["suspects"][0]["category"] == GPU_ISSUE
    assert rep["evidence"]
    dropped = {e["rank"] for e in rep["exonerated"]}
    assert 2 in dropped and 1 not in dropped
    for e in rep["exonerated"]:
        assert any(u["onset_ms"] <= e["onset_ms"] and u["rank"] != e["rank"]
                   for u in rep["suspects"])
    ref = oracle_or_none()
    if ref:
        assert rep == ref.analyze(topo, prog, cfg, recs, trig, 1)


def test_clean_window_false_trigger(eng):
    topo, prog, cfg = fx.fig5()
    recs = concat(*[completion(r, 0, 0, 400, 450) for r in (1, 2, 3)],
                  completion(2, 1, 1, 455, 470), completion(4, 1, 2, 455, 470))
    rep = eng.analyze_failure(eng.TraceStore(records=recs), eng.Model(topo, prog), cfg,
                              TriggerEvent(FAILURE, 2, 600.0))
    assert rep["verdict"] == V_FALSE and rep["suspects"] == []
    assert rep["records_scanned"] == len(recs)


def test_whole_group_stall_exonerated_upstream(eng):
    topo, prog, cfg, recs = fx.two_group()
    rep = eng.analyze_failure(eng.TraceStore(records=recs), eng.Model(topo, prog), cfg,
                              TriggerEvent(FAILURE, 2, 900.0))
    assert rep["verdict"] == V_SUSPECTS
    assert [s["rank"] for s in rep["suspects"]] == [0]
    dropped = {e["rank"] for e in rep["exonerated"]}
    assert {2, 3} <= dropped
    ref = oracle_or_none()
    if ref:
        assert rep == ref.analyze(topo, prog, cfg, recs, TriggerEvent(FAILURE, 2, 900.0), 1)


def _strag(eng, fix, t, k=None):
    cfg = fix.cfg if k is None else AnalysisConfig(delta_ms=fix.cfg.delta_ms,
                                                   consecutive_iterations_k=k)
    recs = fix.store()
    trig = TriggerEvent(STRAGGLER, 0, t)
    rep = eng.analyze_straggler(eng.TraceStore(records=recs), eng.Model(fix.topo, fix.prog),
                                cfg, trig)
    ref = oracle_or_none()
    if ref:
        assert rep == ref.analyze(fix.topo, fix.prog, cfg, recs, trig, 2)
    return rep


def test_constant_late_start(eng):
    fix = fx.Straggler()
    for j in range(4):
        fix.add_iteration(j, 0, 50, 1250)
    rep = _strag(eng, fix, 40000.0)
    assert rep["verdict"] == V_SUSPECTS
    assert [(s["rank"], s["category"]) for s in rep["suspects"]] == [(2, LATE_START)]
    shifted = fx.Straggler()
    for j in range(4):
        shifted.add_iteration(j, 0, 50, 1250, 5000.0)
    r2 = _strag(eng, shifted, 45000.0)
    assert [(s["rank"], s["category"]) for s in r2["suspects"]] == [(2, LATE_START)]


def test_tight_group_no_straggler(eng):
    fix = fx.Straggler()
    for j in range(4):
        fix.add_iteration(j, 0, 30, 50)
    fix.recs.append(state(0, 0, 4, 39990, 1, 1, 1))
    assert _strag(eng, fix, 40000.0)["verdict"] == V_NOSTRAG


def test_nonconstant_lateness(eng):
    fix = fx.Straggler()
    fix.add_iteration(0, 0, 50, 1250)
    fix.add_iteration(1, 0, 50, 60)
    fix.add_iteration(2, 0, 50, 1250)
    fix.add_iteration(3, 0, 50, 1250)
    fix.recs.append(state(0, 0, 4, 39990, 1, 1, 1))
    assert _strag(eng, fix, 40000.0, k=4)["verdict"] == V_NOSTRAG


def test_flow_skew(eng):
    fix = fx.Straggler()
    for j in range(3):
        fix.add_iteration(j, 0, 10, 20)
    base = 30000.0
    fix.recs.append(completion(0, 0, 3, base, base + 30))
    fix.recs.append(completion(2, 0, 3, base, base + 30))
    for ch in range(4):
        fix.recs.append(completion(1, 0, 3, base, base + (75 if ch == 2 else 30), ch))
    fix.recs.append(state(0, 0, 4, 39990, 1, 1, 1))
    rep = _strag(eng, fix, 40000.0)
    assert rep["verdict"] == V_SUSPECTS
    assert [(s["rank"], s["category"]) for s in rep["suspects"]] == [(1, FLOW_SKEWED)]


def test_insufficient_history(eng):
    fix = fx.Straggler()
    fix.add_iteration(0, 0, 50, 1250)
    fix.add_iteration(1, 0, 50, 1250)
    fix.recs.append(state(0, 0, 2, 19990, 1, 1, 1))
    assert _strag(eng, fix, 20000.0)["verdict"] == V_INSUFF


def test_analysis_config_validated(eng):
    topo, prog, _ = fx.fig5()
    with pytest.raises(eng.EngineError) as e:
        eng.analyze_failure(eng.TraceStore(records=fx.fig5_slow_gpu1()),
                            eng.Model(topo, prog), AnalysisConfig(flow_skew_factor=1.0),
                            TriggerEvent(FAILURE, 4, 800.0))
    assert e.value.status == 2
    assert e.value.msg == "analysis: flow_skew_factor must be > 1"


def test_rc_table_invariant_raises_data_error(eng):
    """TraceStore::append does not validate, so a bad state sum reaches
    check_rc_table, which throws DataError (status 4)."""
    topo, prog, cfg = fx.fig5()
    recs = concat(state(1, 0, 3, 600, 1, 2, 0), state(2, 0, 3, 600, 5, 5, 5),
                  state(3, 0, 3, 600, 5, 5, 5))
    with pytest.raises(eng.EngineError) as e:
        eng.analyze_failure(eng.TraceStore(records=recs), eng.Model(topo, prog), cfg,
                            TriggerEvent(FAILURE, 1, 800.0))
    assert e.value.status == 4
    assert "check_rc_table" in e.value.msg
