"""Device JSONL ingest (csrc/jsonl.cu, csrc/jsonl.cuh).

CPU tests pin the host instantiation of the device line parser and of its
decimal -> binary64 conversion (the same __host__ __device__ code the kernel
runs): doubles bit-identical to Python's correctly rounded float() on random
and adversarial tokens, lines identical to the reference's packing, and every
line the exact parser rejects rejected (deferred) here too. GPU tests run the
ingest kernels on whole traces and through collsight_run_analyze."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import GOLDEN, ROOT
from tests.test_jsonl import VARIANTS, _exact


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _check_double(eng, tok: str):
    got = eng.jsonl_parse_double(tok)
    want = float(tok)
    if got is None:  # deferred: only subnormal / overflow / > 19 digits / "-0"
        return False
    assert bits(got) == bits(want), (tok, got, want)
    return True


def test_double_shortest_reprs(eng):
    """repr() of random doubles over the whole exponent range (the simulator
    writes std::to_chars shortest forms)."""
    rng = np.random.default_rng(1)
    raw = rng.integers(0, 2**63, 20000, dtype=np.uint64)
    vals = raw.view(np.float64)
    n = 0
    for v in vals:
        if not np.isfinite(v) or v == 0 or abs(v) < 2.3e-308:
            continue
        for tok in (repr(float(v)), repr(-float(v)), "%.17g" % v, "%.15e" % v):
            n += _check_double(eng, tok)
    assert n > 70000


def test_double_decimal_grid(eng):
    """Random decimal strings of 1-19 digits with exponents across the
    normal range, in fixed and scientific notation."""
    rng = np.random.default_rng(2)
    accepted = 0
    for _ in range(40000):
        nd = int(rng.integers(1, 20))
        digits = "".join(str(int(d)) for d in rng.integers(0, 10, nd))
        e = int(rng.integers(-320, 300))
        tok = f"{digits}e{e}"
        accepted += _check_double(eng, tok)
        k = int(rng.integers(0, nd + 1))
        tok2 = (digits[:k] or "0") + "." + (digits[k:] or "0")
        if tok2[0] == "0" and len(tok2) > 1 and tok2[1] != ".":
            tok2 = tok2.lstrip("0") or "0"
            if tok2.startswith("."):
                tok2 = "0" + tok2
        accepted += _check_double(eng, tok2)
    assert accepted > 70000


def test_double_halfway_and_edges(eng):
    """Ties to even, the Clinger bound, the refinement branch, powers of ten
    at the table ends; subnormals / overflow / 20 digits defer."""
    toks = ["9007199254740993", "9007199254740995", "9007199254740992",
            "18014398509481985", "1e23", "8.98846567431158e307",
            "1.7976931348623157e308", "2.2250738585072014e-308", "4.9e-324",
            "1.7976931348623159e308", "0.1", "0.30000000000000004", "123456789012345678",
            "1234567890123456789", "12345678901234567890", "5e-324", "1e-342", "1e308",
            "2.5", "3.5", "0.5e1", "1E22", "1e22", "9.999999999999999e22", "1.0e-5",
            "0.000001", "-0.0", "-0", "0", "0.0", "-1.5e-7", "4503599627370496.5",
            "4503599627370497.5", "2.2250738585072011e-308",
            "7.2057594037927933e16", "7.2057594037927936e16"]
    for t in toks:
        _check_double(eng, t)
    assert eng.jsonl_parse_double("4.9e-324") is None      # subnormal
    assert eng.jsonl_parse_double("1.8e308") is None       # overflow
    assert eng.jsonl_parse_double("12345678901234567890") is None  # 20 digits
    assert eng.jsonl_parse_double("-0") is None            # integer -0
    got = eng.jsonl_parse_double("-0.0")
    assert got == 0.0 and bits(got) == bits(-0.0)
    # ties: 2^53 + 1 rounds to even (2^53), 2^53 + 3 to 2^53 + 4
    assert eng.jsonl_parse_double("9007199254740993") == 9007199254740992.0
    assert eng.jsonl_parse_double("9007199254740995") == 9007199254740996.0


def _catalog_text(oracle, name):
    cfg = open(os.path.join(GOLDEN, "configs", f"{name}.json")).read()
    return oracle.simulate(cfg, with_jsonl=True)


@pytest.mark.parametrize("name", ["scenario1", "scenario7"])
def test_lines_match_reference_packing(eng, oracle, name):
    recs, text = _catalog_text(oracle, name)
    lines = text.splitlines()
    assert len(lines) == len(recs)
    # (bytes, not np.concatenate: the record dtype's union fields overlap)
    got = b"".join(eng.jsonl_parse_line(l).tobytes() for l in lines)
    assert got == recs.tobytes()


def _exact_lines(lines):
    """Per line: the exact parser's record bytes, or None if it rejects the
    line (one child process, CSG_JSONL_EXACT=1)."""
    code = ("import sys, json; sys.path.insert(0, %r);"
            "from paper_2509_03018_b200 import engine as E;"
            "out = []\n"
            "for l in json.load(sys.stdin):\n"
            "    try:\n"
            "        out.append(E.parse_trace(l + '\\n').tobytes().hex())\n"
            "    except E.EngineError:\n"
            "        out.append(None)\n"
            "json.dump(out, sys.stdout)" % ROOT)
    env = dict(os.environ, CSG_JSONL_EXACT="1")
    r = subprocess.run([sys.executable, "-c", code], input=json.dumps(lines).encode(),
                       env=env, capture_output=True, timeout=600)
    assert r.returncode == 0, r.stderr.decode()[-2000:]
    return [bytes.fromhex(h) if h is not None else None for h in json.loads(r.stdout)]


@pytest.mark.parametrize("k", range(len(VARIANTS)))
def test_mutated_lines_never_accepted_wrongly(eng, oracle, k):
    """A line is accepted only with the exact parser's record; every line the
    exact parser rejects is deferred."""
    _, text = _catalog_text(oracle, "clean")
    muts = [VARIANTS[k](l) for l in text.splitlines()[:400:20]]
    for m, want in zip(muts, _exact_lines(muts)):
        rec = eng.jsonl_parse_line(m)
        if want is None:
            assert rec is None, m
        elif rec is not None:
            assert rec.tobytes() == want, m


def test_field_order_and_whitespace_take_the_general_path(eng, oracle):
    """Lines in the serializer's field order go through the register-only
    fast path; any other order or spacing goes through the general parser.
    Both must give the reference's record."""
    recs, text = _catalog_text(oracle, "scenario1")
    rng = np.random.default_rng(7)
    lines = text.splitlines()
    for i in rng.choice(len(lines), size=300, replace=False):
        obj = json.loads(lines[i])
        keys = list(obj)
        rng.shuffle(keys)
        for sep in ((",", ":"), (", ", ": ")):
            l = json.dumps({k: obj[k] for k in keys}, separators=sep)
            # json.dumps writes floats with repr(): the same shortest digits
            got = eng.jsonl_parse_line(l)
            assert got is not None, l
            assert got.tobytes() == recs[i:i + 1].tobytes(), l


def test_short_and_odd_lines_defer(eng):
    for l in ["", " ", "{}", "[]", '{"type":"state"}', "{" * 200, '"x"', "\r",
              '{"type":"completion","node":0,"comm_id":0,"rank":0,"channel":0,'
              '"op_seq":0,"op_name":"Bcast","msg_bytes":1,"start_ms":0,"end_ms":0}']:
        assert eng.jsonl_parse_line(l) is None, l


# ---------------------------------------------------------------- GPU
def _ingest_child(text_path: str, env: dict) -> bytes:
    code = ("import sys; sys.path.insert(0, %r);"
            "from paper_2509_03018_b200 import engine as E;"
            "s = E.TraceStore();"
            "ok = s.append_jsonl_file(%r);"
            "sys.stdout.buffer.write((b'OK' if ok else b'NO') + s.records().tobytes())"
            % (ROOT, text_path))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                       capture_output=True, timeout=600)
    assert r.returncode == 0, r.stderr.decode()[-2000:]
    return r.stdout


@pytest.mark.gpu
def test_device_ingest_matches_reference(eng, oracle):
    recs, text = _catalog_text(oracle, "scenario7")
    store = eng.TraceStore()
    assert store.append_jsonl(text)
    assert store.records().tobytes() == recs.tobytes()
    # appends after existing records, no trailing newline, CRLF line ends
    assert store.append_jsonl(text.rstrip("\n").replace("\n", "\r\n"))
    assert store.records().tobytes() == recs.tobytes() * 2


@pytest.mark.gpu
def test_device_ingest_small_chunks_and_super_chunks(eng, oracle, tmp_path):
    """64 KB staging chunks and 1 MB device super-chunks (cut at newlines)."""
    recs, text = _catalog_text(oracle, "scenario1")
    p = tmp_path / "t.jsonl"
    p.write_text(text * 3)
    out = _ingest_child(str(p), {"CSG_JSONL_CHUNK_KB": "64", "CSG_JSONL_SUPER_MB": "1"})
    assert out[:2] == b"OK"
    assert out[2:] == recs.tobytes() * 3


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(VARIANTS)))
def test_device_ingest_defers_on_edge_lines(eng, oracle, k, tmp_path):
    _, text = _catalog_text(oracle, "clean")
    lines = text.splitlines()
    rng = np.random.default_rng(k)
    for i in rng.choice(len(lines), size=3, replace=False):
        lines[i] = VARIANTS[k](lines[i])
    mutated = "\n".join(lines) + "\n"
    store = eng.TraceStore()
    ok = store.append_jsonl(mutated)
    exact = _exact(mutated)
    if ok:
        assert store.records().tobytes() == exact
    else:
        assert len(store) == 0
    # the drop-in call: same status/message or same reports as the exact path
    p = tmp_path / "m.jsonl"
    p.write_text(mutated)
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", "clean.json"))
    try:
        got = eng.run_analyze(scen, str(p)).reports_jsonl
    except eng.EngineError as e:
        got = ("ERR %d %s" % (e.status, e.msg))
    if exact.startswith(b"ERR"):
        assert got == exact.decode()
    else:
        assert not got.startswith("ERR")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scenario1", "scenario3", "scenario7", "sweep_opseq_lag"])
def test_run_analyze_file_matches_reference(eng, name, tmp_path):
    """collsight_run_analyze on a JSONL trace (device ingest) reproduces the
    reference's reports_to_jsonl bytes."""
    from tests.test_gpu_catalog import golden
    recs, reports, _ = golden(name)
    text = eng.serialize_records(recs)
    p = tmp_path / "t.jsonl"
    p.write_text(text)
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
    res = eng.run_analyze(scen, str(p))
    assert res.reports_jsonl == reports
    store = eng.TraceStore()
    assert store.append_jsonl_file(str(p))
    assert store.records().tobytes() == recs.tobytes()
