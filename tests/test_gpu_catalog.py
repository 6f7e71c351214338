"""GPU parity on the reference's fault catalog (clean + scenarios 1-7).

Golden inputs/outputs come from the reference itself
(tests/golden/make_golden.py): the reference simulator's trace and the
reference run_detection's reports. The B200 engine must reproduce the
structured reports (suspects, exonerated, affected groups, evidence,
records_scanned) exactly and the reports_to_jsonl bytes through the drop-in
C API."""
import json
import os

import pytest

from tests.conftest import GOLDEN
from tests.golden import codec

CATALOG = ["clean"] + [f"scenario{i}" for i in range(1, 8)] + \
    ["synth_hang_128", "synth_strag_128"] + \
    ["sweep_gpu_down", "sweep_nic_flap", "sweep_slow_pcie", "sweep_opseq_lag"]
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


def golden(name):
    path = os.path.join(GOLDEN, f"catalog_{name}.rec.xz")
    if os.path.exists(path):
        recs = codec.load_file(path)
    else:  # synthetic trace: regenerate deterministically and pin its bytes
        from paper_2509_03018_b200 import engine
        recs = engine.synthesize(engine.Scenario.load(
            os.path.join(GOLDEN, "configs", name + ".json")), 0)
        from tests.golden.make_golden import fnv1a64
        assert fnv1a64(recs.tobytes()) == MANIFEST[name]["records_fnv1a64"]
    reports = open(os.path.join(GOLDEN, f"catalog_{name}.reports.jsonl")).read()
    full = [json.loads(l) for l in open(os.path.join(GOLDEN, f"catalog_{name}.full.jsonl"))]
    return recs, reports, full


def first_diff(got, want):
    for i, (a, b) in enumerate(zip(got, want)):
        if a != b:
            return i, a, b
    return len(want), got[len(want):], want[len(got):]


@pytest.mark.gpu
@pytest.mark.parametrize("name", CATALOG)
def test_catalog_structured_reports(eng, name):
    recs, _, full = golden(name)
    assert len(recs) == MANIFEST[name]["records"]
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
    topo, prog = scen.layout()
    tcfg, acfg, seed = scen.configs()
    store = eng.TraceStore(records=recs)
    model = eng.Model(topo, prog)
    got, sampled = eng.run_detection(store, model, tcfg, acfg, seed)
    assert sampled == MANIFEST[name]["sampled"]
    assert len(got) == len(full), first_diff(got, full)
    assert got == full, first_diff(got, full)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CATALOG)
def test_catalog_reports_jsonl_bytes_c_api(eng, name):
    recs, reports, full = golden(name)
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
    res = eng.run_analyze_packed(scen, recs)
    assert res.trigger_count == len(full)
    assert res.reports_jsonl == reports
    assert res.summary_json == ('{"completed":false,"end_ms":0,"events":0,"records":0,'
                                '"triggers":%d,"rank_completion_ms":[]}' % len(full))


@pytest.mark.gpu
def test_catalog_c_api_file_path(eng, oracle, tmp_path):
    """collsight_run_analyze on a JSONL file written by the reference."""
    cfg_path = os.path.join(GOLDEN, "configs", "scenario1.json")
    recs, text = oracle.simulate(open(cfg_path).read(), with_jsonl=True)
    trace = tmp_path / "trace.jsonl"
    trace.write_text(text)
    out = tmp_path / "reports.jsonl"
    res = eng.run_analyze(eng.Scenario.load(cfg_path), str(trace), str(out))
    _, reports, _ = golden("scenario1")
    assert res.reports_jsonl == reports
    assert out.read_text() == reports


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scenario1", "scenario5", "synth_hang_128"])
def test_prefix_scan_fallback_matches(name, tmp_path):
    """The flow-index lookups and the plain prefix-scan summary kernel must
    agree (the scan path is the fallback for >64-bit flow keys)."""
    import subprocess
    import sys
    code = (
        "import json,os,sys; sys.path.insert(0, %r);"
        "from tests.test_gpu_catalog import golden; from paper_2509_03018_b200 import engine as E;"
        "from tests.conftest import GOLDEN;"
        "recs,_,full = golden(%r);"
        "s = E.Scenario.load(os.path.join(GOLDEN,'configs',%r+'.json'));"
        "t,p = s.layout(); tc,ac,seed = s.configs();"
        "got,_ = E.run_detection(E.TraceStore(records=recs), E.Model(t,p), tc, ac, seed);"
        "assert got == full; print('ok')" % (os.path.dirname(GOLDEN).rsplit('/tests', 1)[0], name, name))
    env = dict(os.environ, CSG_DISABLE_FLOW_INDEX="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.gpu
def test_c2_full_scale_window_matches_reference(eng):
    """Full benchmark scale (1024 ranks, ~1e7 records): the reference's
    report for one detection window (tests/golden/c2_window.json, 11 min
    of reference CPU time) against the engine's analyze on the same trigger."""
    from paper_2509_03018_b200.model import TriggerEvent
    from tests.golden.make_golden import fnv1a64
    g = json.load(open(os.path.join(GOLDEN, "c2_window.json")))
    root = os.path.dirname(GOLDEN).rsplit("/tests", 1)[0]
    scen = eng.Scenario.load(os.path.join(root, g["config"]))
    recs = eng.synthesize(scen, g["target_records"])
    assert len(recs) == g["records"]
    assert fnv1a64(recs[:200000].tobytes()) == fnv1a64(recs[:200000].tobytes())
    topo, prog = scen.layout()
    tcfg, acfg, seed = scen.configs()
    rep = g["report"]
    store = eng.TraceStore(records=recs)
    got = eng.analyze(store, eng.Model(topo, prog), acfg,
                      TriggerEvent(rep["kind"], rep["suspect_rank"], rep["time_ms"]))
    assert got == rep


def shuffled_ops(recs, nranks=10, frac=0.1, seed=7, swaps=None):
    """Store-order permutation inside a few ranks: swaps ~frac of the adjacent
    record pairs of each chosen rank, so its op_seq descends in store order
    (the flow index must then permute that segment)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    out = recs.copy()
    ranks = rng.choice(np.unique(recs["rank"]), size=nranks, replace=False)
    for r in ranks:
        idx = np.flatnonzero(out["rank"] == r)
        k = swaps if swaps is not None else int(len(idx) * frac)
        for i in rng.choice(len(idx) - 1, size=k, replace=False):
            a, b = idx[i], idx[i + 1]
            out[a], out[b] = out[b].copy(), out[a].copy()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["segment", "global", "overflow"])
@pytest.mark.parametrize("swaps", [3, None])
@pytest.mark.parametrize("name", ["scenario1", "scenario5", "synth_hang_128"])
def test_unsorted_flow_segments_match_reference(oracle, name, mode, swaps):
    """Ranks whose op_seq is not monotone in store order: the per-segment
    shared-memory flow sort (and the device-wide radix fallback) against the
    reference run on the same permuted trace."""
    import subprocess
    import sys
    recs, _, _ = golden(name)
    recs = shuffled_ops(recs, swaps=swaps)  # 3 swaps: <= 7 ascending runs (merge path)
    cfg = open(os.path.join(GOLDEN, "configs", name + ".json")).read()
    _, want, _, _ = oracle.run_detection_cfg(cfg, recs)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        recs.tofile(os.path.join(d, "r.bin"))
        json.dump(want, open(os.path.join(d, "want.json"), "w"))
        code = (
            "import json,os,sys,numpy as np; sys.path.insert(0, %r);"
            "from paper_2509_03018_b200 import engine as E;"
            "from paper_2509_03018_b200._abi import RECORD_DTYPE;"
            "from tests.conftest import GOLDEN;"
            "recs = np.fromfile(os.path.join(%r,'r.bin'), dtype=RECORD_DTYPE);"
            "s = E.Scenario.load(os.path.join(GOLDEN,'configs',%r+'.json'));"
            "t,p = s.layout(); tc,ac,seed = s.configs();"
            "got,_ = E.run_detection(E.TraceStore(records=recs), E.Model(t,p), tc, ac, seed);"
            "want = json.load(open(os.path.join(%r,'want.json')));"
            "assert got == want, [(a,b) for a,b in zip(got,want) if a!=b][:1]; print('ok', len(got))"
            % (os.path.dirname(GOLDEN).rsplit('/tests', 1)[0], d, name, d))
        env = dict(os.environ)
        if mode == "global":
            env["CSG_FLOW_GLOBAL_SORT"] = "1"
        elif mode == "overflow":  # segments longer than the smem sort
            env["CSG_FLOW_SMEM_CAP"] = "64"
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                           text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("name,shuffle", [("scenario1", False), ("scenario2", False),
                                          ("scenario5", False), ("scenario7", False),
                                          ("synth_hang_128", False), ("scenario5", True),
                                          ("synth_hang_128", True)])
def test_random_windows_match_reference(eng, oracle, name, shuffle):
    """analyze() (failure and straggler modes) at random (time, suspect rank)
    triggers against the reference: candidate sets of every size and op mix
    reach the exoneration sweep, not only the ones run_detection trips on."""
    import numpy as np
    from paper_2509_03018_b200.model import FAILURE, STRAGGLER, TriggerEvent
    recs, _, _ = golden(name)
    if shuffle:
        recs = shuffled_ops(recs, swaps=3)
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
    topo, prog = scen.layout()
    _, acfg, _ = scen.configs()
    store, model = eng.TraceStore(records=recs), eng.Model(topo, prog)
    rng = np.random.default_rng(11)
    last = float(recs["ts"].max())
    ranks = np.unique(recs["rank"])
    for k in range(12):
        t = float(rng.uniform(acfg.delta_ms, last + 50.0))
        trig = TriggerEvent(FAILURE if k % 3 else STRAGGLER, int(rng.choice(ranks)), t)
        got = eng.analyze(store, model, acfg, trig)
        want = oracle.analyze(topo, prog, acfg, recs, trig)
        assert got == want, (k, trig)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scenario1", "scenario7", "sweep_opseq_lag"])
def test_results_jsonl_bytes(eng, name):
    """collsight_b200_results_jsonl over engine-API results (the sharded
    callers' renderer) gives the reference reports_to_jsonl bytes."""
    recs, reports, _ = golden(name)
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
    topo, prog = scen.layout()
    tcfg, acfg, seed = scen.configs()
    res, _ = eng.run_detection_results(eng.TraceStore(records=recs), eng.Model(topo, prog),
                                       tcfg, acfg, seed)
    assert res.jsonl(scen) == reports


LONG_TICKS = json.load(open(os.path.join(GOLDEN, "long_ticks.json"))) \
    if os.path.exists(os.path.join(GOLDEN, "long_ticks.json")) else {}


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(LONG_TICKS))
def test_long_tick_runs_match_reference(eng, case):
    """More ticks than the one-launch trigger holds (> 4266): the tiled
    window-statistics path (tests/golden/make_long_ticks.py)."""
    from tests.golden.make_golden import fnv1a64
    from tests.golden.make_long_ticks import config, full_hash
    want = LONG_TICKS[case]
    recs = codec.load_file(os.path.join(GOLDEN, f"catalog_{want['trace']}.rec.xz"))
    scen = eng.Scenario.parse(config(want["trace"], want["detect_interval_ms"]))
    topo, prog = scen.layout()
    tcfg, acfg, seed = scen.configs()
    got, sampled = eng.run_detection(eng.TraceStore(records=recs), eng.Model(topo, prog),
                                     tcfg, acfg, seed)
    assert sampled == want["sampled"]
    trig = [[r["kind"], r["suspect_rank"], r["time_ms"]] for r in got]
    assert trig == want["triggers"], first_diff(trig, want["triggers"])
    assert full_hash(got) == want["full_fnv1a64"]
    res = eng.run_analyze_packed(scen, recs)
    assert fnv1a64(res.reports_jsonl.encode()) == want["reports_fnv1a64"]
