"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every function include/*.h declares, and its host-side pieces (table
functions, layout/program builder, scenario + trace parsers) agree with the
reference. No device calls."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT

HEADERS = ["csg_engine.h", "collsight.h", "collsight_b200.h"]


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:csg|collsight)_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol(eng):
    lib = eng.lib()
    names = [n for h in HEADERS for n in declared(h)]
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_native():
    so = os.path.join(ROOT, "paper_2509_03018_b200", "lib", "libcollsight_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_versions(eng):
    assert eng.lib().collsight_version().decode() == "0.1.0"


# --- Table functions (proj/tests/test_rca.cpp:102-210) ----------------------

def test_check_min_op_kats(eng, oracle):
    assert eng.check_min_op([(0, 42), (1, 41), (2, 42), (3, 42)]) == [1]
    assert eng.check_min_op([(0, 42), (1, 42), (2, 42)]) is None
    assert eng.check_min_op([(5, 7), (2, 3), (9, 3)]) == [2, 9]
    with pytest.raises(eng.EngineError):
        eng.check_min_op([])
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(1, 9))
        pairs = [(int(r), int(rng.integers(0, 4))) for r in rng.permutation(20)[:n]]
        assert eng.check_min_op(pairs) == oracle.check_min_op(pairs)


def test_check_min_data_kats(eng, oracle):
    pairs = [(0, (5, 5, 5)), (1, (5, 4, 4)), (2, (5, 5, 3))]
    assert eng.check_min_data(pairs) == oracle.check_min_data(pairs) == [2]
    uni = [(3, (2, 2, 2)), (1, (2, 2, 2))]
    assert eng.check_min_data(uni) == [1, 3]
    rng = np.random.default_rng(11)
    for _ in range(200):
        n = int(rng.integers(1, 7))
        pairs = []
        for r in rng.permutation(30)[:n]:
            d = int(rng.integers(0, 3)); t = d + int(rng.integers(0, 2))
            pairs.append((int(r), (t + int(rng.integers(0, 2)), t, d)))
        assert eng.check_min_data(pairs) == oracle.check_min_data(pairs)


def test_rc_table_totality(eng, oracle):
    # Table 4 totality: 56 cells 0 <= done <= tx <= staged <= 5
    cells = 0
    for staged in range(6):
        for tx in range(staged + 1):
            for done in range(tx + 1):
                if staged + tx + done == 0 or True:
                    c = (staged, tx, done)
                    assert eng.check_rc_table(c) == oracle.check_rc_table(c)
                    for peer in [(5, 5, 5), (5, 5, 3), (4, 2, 1)]:
                        assert eng.check_rc_table(c, peer) == oracle.check_rc_table(c, peer)
                    cells += 1
    assert cells == 56
    # remote cross-check (5,5,3) vs (5,5,5) -> (ReceiverFailed, Remote)
    assert eng.check_rc_table((5, 5, 3), (5, 5, 5)) == (2, 1)
    with pytest.raises(eng.EngineError) as e:
        eng.check_rc_table((1, 2, 0))
    assert e.value.status == 4


# --- layout / program -------------------------------------------------------

@pytest.mark.parametrize("shape", [(8, 2, 2, 8, 2, 4), (1, 1, 32, 1, 4, 4),
                                   (4, 3, 2, 4, 2, 2), (2, 1, 2, 2, 1, 4),
                                   (8, 4, 32, 8, 4, 4), (1, 1, 1, 1, 1, 1),
                                   (2, 4, 1, 2, 1, 1)])
def test_layout_and_program_match_reference(eng, oracle, shape):
    t1, p1 = eng.build_layout(*shape)
    t2, p2 = oracle.layout(*shape)
    assert t1 == t2
    assert p1 == p2


# --- scenario + trace parsing (C API error conventions) ---------------------

def _ref_capi():
    L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libcollsight_ref.so"))
    L.collsight_last_error.restype = C.c_char_p
    return L


BAD_CONFIGS = [
    '{"layout":{}}',
    'not json',
    '[1,2]',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1}',
    '{"layout":{"tp":4,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"trigger":{"ema_alpha":0}}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"analysis":{"flow_skew_factor":1}}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"faults":{}}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"faults":[{"kind":"zap","onset_ms":1,"node":0}]}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"faults":[{"kind":"nic_shutdown","onset_ms":1,"nic":0}]}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"faults":[{"kind":"nic_shutdown","onset_ms":1,"node":3}]}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"sim":{"chunk_bytes":0}}',
    '{"layout":{"tp":2,"pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1,"msg_bytes":0}',
    '{"layout":{"tp":"x","pp":1,"dp":1,"ranks_per_node":2,"channels_per_pair":1},"iterations":1,"seed":1}',
]


@pytest.mark.parametrize("text", BAD_CONFIGS)
def test_scenario_errors_match_reference(eng, oracle, text):
    R = _ref_capi()
    h = C.c_void_p()
    st_ref = R.collsight_scenario_parse(text.encode(), C.byref(h))
    msg_ref = R.collsight_last_error().decode()
    with pytest.raises(eng.EngineError) as e:
        eng.Scenario.parse(text)
    assert (e.value.status, e.value.msg) == (st_ref, msg_ref)


def test_scenario_null_argument(eng):
    L = eng.lib()
    assert L.collsight_scenario_parse(None, None) == 5
    assert L.collsight_last_error().decode() == "null argument"
    assert L.collsight_run_analyze(None, None, None, None) == 5


def test_catalog_configs_parse_like_reference(eng):
    from tests.conftest import GOLDEN
    for name in ["clean"] + [f"scenario{i}" for i in range(1, 8)]:
        s = eng.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
        t, a, seed = s.configs()
        assert seed == 42 and t.max_sampled_ranks == 16
        assert a.delta_ms == t.delta_ms


BAD_LINES = [
    '{"type":"completion"}',
    'garbage',
    '[1]',
    '{"type":"x"}',
    '{"type":"state","node":0,"comm_id":0,"rank":0,"channel":0,"op_seq":0,"window_end_ms":1,"stuck_ms":0,"total_chunks":1,"gpu_ready":2,"rdma_transmitted":0,"rdma_done":0}',
    '{"type":"completion","node":0,"comm_id":0,"rank":0,"channel":0,"op_seq":0,"op_name":"AllGather","msg_bytes":1,"start_ms":5,"end_ms":4}',
    '{"type":"completion","node":0,"comm_id":0,"rank":0,"channel":0,"op_seq":0,"op_name":"Bcast","msg_bytes":1,"start_ms":1,"end_ms":4}',
    '{"type":"completion","node":0,"comm_id":0,"rank":-1,"channel":0,"op_seq":0,"op_name":"Send","msg_bytes":1,"start_ms":1,"end_ms":4}',
    '{"type":"completion","node":0,"comm_id":0,"rank":1,"channel":0,"op_seq":0,"op_name":"Send","msg_bytes":0,"start_ms":1,"end_ms":4}',
    '{"type":"completion","node":0,"comm_id":0,"rank":1,"channel":0,"op_seq":0,"op_name":"Send","msg_bytes":1,"start_ms":1,"end_ms":4,"extra":1}',
]


@pytest.mark.parametrize("line", BAD_LINES)
def test_trace_parse_errors_match_reference(eng, oracle, tmp_path, line):
    path = tmp_path / "t.jsonl"
    path.write_text('\n' + line + '\n')
    R = _ref_capi()
    cfg = open(os.path.join(ROOT, "tests", "golden", "configs", "clean.json")).read()
    h = C.c_void_p()
    assert R.collsight_scenario_parse(cfg.encode(), C.byref(h)) == 0
    res = C.c_void_p()
    st_ref = R.collsight_run_analyze(h, str(path).encode(), None, C.byref(res))
    msg_ref = R.collsight_last_error().decode()
    s = eng.Scenario.parse(cfg)
    with pytest.raises(eng.EngineError) as e:
        eng.run_analyze(s, str(path))
    assert (e.value.status, e.value.msg) == (st_ref, msg_ref)


def test_missing_trace_file(eng):
    cfg = open(os.path.join(ROOT, "tests", "golden", "configs", "clean.json")).read()
    s = eng.Scenario.parse(cfg)
    with pytest.raises(eng.EngineError) as e:
        eng.run_analyze(s, "/nonexistent.jsonl")
    assert e.value.status == 3
    assert e.value.msg == "line 0: cannot open trace file '/nonexistent.jsonl'"


def test_jsonl_roundtrip_matches_reference_packing(eng, oracle):
    cfg = open(os.path.join(ROOT, "tests", "golden", "configs", "scenario3.json")).read()
    recs, text = oracle.simulate(cfg, with_jsonl=True)
    got = eng.parse_trace(text)
    assert got.tobytes() == recs.tobytes()
