"""The straggler self-evidence filter (rca.cpp:795-869) has two device
paths: the sorted-segment warp path (k_opsort + k_sf_fast, the default) and
the per-candidate block path (k_self_faulted) it defers to; the iteration
tables likewise have an incremental one-pass form (default) and a per-trip
form (CSG_ITER_PER_TRIP=1). Both must give
the reference's reports: the catalog tests run the default path against the
reference's golden reports; here the block path alone (CSG_SF_SLOW=1) runs
the same straggler cases, and a C3-shaped fail-slow trace (1024 ranks, 16
channels, three fail-slow faults; thousands of lateness candidates per trip)
must produce identical reports on both paths, also with shuffled store
order inside some ranks (permuted flow segments)."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import GOLDEN

ROOT = os.path.dirname(GOLDEN).rsplit("/tests", 1)[0]

RUN = r"""
import json, sys
sys.path.insert(0, %(root)r)
from paper_2509_03018_b200 import engine as E
from tests.test_gpu_catalog import golden, shuffled_ops
if %(cfg)r.endswith('.json'):
    s = E.Scenario.load(%(cfg)r)
    recs = E.synthesize(s, 0)
else:
    s = E.Scenario.load(%(root)r + '/tests/golden/configs/%(cfg)s.json')
    recs = golden(%(cfg)r)[0]
if %(shuffle)r:
    recs = shuffled_ops(recs, nranks=24, swaps=5)
t, p = s.layout(); tc, ac, seed = s.configs()
got, _ = E.run_detection(E.TraceStore(records=recs), E.Model(t, p), tc, ac, seed)
print(json.dumps(got))
"""


KNOBS = ("CSG_SF_SLOW", "CSG_ITER_PER_TRIP", "CSG_SL_SERIAL", "CSG_FLOW_SCAN",
         "CSG_EXO_WARP_SWEEP")


def run(cfg, slow=False, shuffle=False, per_trip=False):
    """slow: the block-per-candidate self-evidence filter, the per-trip
    iteration tables and the serial (block per trip) candidate generation
    instead of the parallel defaults."""
    env = {k: v for k, v in os.environ.items() if k not in KNOBS}
    if slow:
        env["CSG_SF_SLOW"] = "1"
        env["CSG_SL_SERIAL"] = "1"
        env["CSG_FLOW_SCAN"] = "1"
        env["CSG_EXO_WARP_SWEEP"] = "1"
    if per_trip:
        env["CSG_ITER_PER_TRIP"] = "1"
    code = RUN % {"root": ROOT, "cfg": cfg, "shuffle": shuffle}
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                       text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["synth_strag_128", "scenario5", "scenario7", "scenario1",
                                  "synth_hang_128"])
def test_block_path_matches_reference(name):
    """The per-candidate block filter, the per-trip iteration tables, the
    serial candidate loop and the single-warp exoneration sweep (the paths
    the defaults replace or defer to) against the reference."""
    want = [json.loads(l) for l in open(os.path.join(GOLDEN, f"catalog_{name}.full.jsonl"))]
    assert run(name, slow=True, per_trip=True) == want


@pytest.mark.gpu
@pytest.mark.parametrize("shuffle", [False, True])
def test_c3_shape_paths_agree(shuffle):
    cfg = os.path.join(ROOT, "configs", "c3_mini_1024.json")
    fast = run(cfg, shuffle=shuffle)
    slow = run(cfg, slow=True, per_trip=True, shuffle=shuffle)
    assert fast == slow
    strag = [r for r in fast if r["kind"] == 1]  # straggler trips
    assert strag, "the C3-shaped trace must trip the straggler path"
