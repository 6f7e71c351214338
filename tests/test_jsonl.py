"""Multithreaded JSONL ingest (csrc/host/fast_jsonl.cpp) against the exact
nlohmann-based parser (CSG_JSONL_EXACT=1) and the reference's own packing:
identical records on valid traces of every size (the fast path only runs
multithreaded above 1 MiB), and identical status + message whenever the
exact grammar or a record invariant has to decide (the fast path defers)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _exact(text: str) -> bytes:
    """Records (or 'ERR status msg') from the exact parser in a child process."""
    code = ("import sys; sys.path.insert(0, %r);"
            "from paper_2509_03018_b200 import engine as E;"
            "t = sys.stdin.read()\n"
            "try:\n"
            "    sys.stdout.buffer.write(E.parse_trace(t).tobytes())\n"
            "except E.EngineError as e:\n"
            "    sys.stdout.buffer.write(('ERR %%d %%s' %% (e.status, e.msg)).encode())\n" % ROOT)
    env = dict(os.environ, CSG_JSONL_EXACT="1")
    r = subprocess.run([sys.executable, "-c", code], input=text.encode(), env=env,
                       capture_output=True, timeout=600)
    assert r.returncode == 0, r.stderr.decode()[-2000:]
    return r.stdout


def _fast(eng, text: str) -> bytes:
    try:
        return eng.parse_trace(text).tobytes()
    except eng.EngineError as e:
        return ("ERR %d %s" % (e.status, e.msg)).encode()


def test_large_trace_matches_exact_and_reference(eng, oracle):
    cfg = open(os.path.join(ROOT, "tests", "golden", "configs", "scenario7.json")).read()
    recs, text = oracle.simulate(cfg, with_jsonl=True)
    big = text * 3  # > 1 MiB: the threaded path
    assert len(big) > (1 << 20)
    got = _fast(eng, big)
    assert got == recs.tobytes() * 3
    assert got == _exact(big)


VARIANTS = [
    lambda l: l.replace('"rank":', ' "rank" : '),          # whitespace
    lambda l: l.replace('}', '}\r'),                       # CRLF
    lambda l: l.replace('"node":0', '"node":0.0'),         # float in an int field
    lambda l: l.replace('"stuck_ms":0', '"stuck_ms":-0'),  # integer -0 as a double
    lambda l: l.replace('"type"', '"ty\\u0070e"'),         # escaped key
    lambda l: l.replace('"node":0', '"node":0,"node":1'),  # duplicate key
    lambda l: l.replace('"node":0', '"node":9999999999'),  # out of int32 range
    lambda l: l.replace('"gpu_ready":', '"gpu_ready":-'),  # negative counter
    lambda l: l.replace('{', '{"zzz":1,'),                 # unknown field
    lambda l: l.replace('"window_end_ms":', '"window_end_ms":1e3,"x":'),
    lambda l: l[:-2],                                      # truncated
    lambda l: ' ',                                         # blank but not empty
]


@pytest.mark.parametrize("k", range(len(VARIANTS)))
def test_edge_lines_defer_to_the_exact_parser(eng, oracle, k):
    cfg = open(os.path.join(ROOT, "tests", "golden", "configs", "clean.json")).read()
    _, text = oracle.simulate(cfg, with_jsonl=True)
    lines = text.splitlines()
    rng = np.random.default_rng(k)
    for i in rng.choice(len(lines), size=3, replace=False):
        lines[i] = VARIANTS[k](lines[i])
    mutated = "\n".join(lines) + "\n"
    assert len(mutated) > (1 << 20)  # the threaded path
    assert _fast(eng, mutated) == _exact(mutated)
    head = "\n".join(lines[:2000]) + "\n"  # under 1 MiB: single-threaded
    assert _fast(eng, head) == _exact(head)
