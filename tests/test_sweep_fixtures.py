"""C5 fault-injection sweep fixtures (tests/golden/make_sweep.py) pinned to
the reference: each case's trace is regenerated through the reference
simulator (+ the deterministic record-level edit) and must hash to the
committed fixture, and the reference run_detection over it must reproduce the
committed reports_to_jsonl bytes. The GPU parity over these fixtures runs in
tests/test_gpu_catalog.py (1 GPU) and tests/test_gpu_multi.py (sharded)."""
import json
import os

import pytest

from tests.conftest import GOLDEN
from tests.golden import codec
from tests.golden.make_sweep import CASES

MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


@pytest.mark.parametrize("name", CASES)
def test_sweep_fixture_pinned_to_reference(oracle, name):
    from tests.golden.make_golden import fnv1a64
    from tests.golden.make_sweep import case
    _, recs = case(name)
    assert fnv1a64(recs.tobytes()) == MANIFEST[name]["records_fnv1a64"]
    assert (recs == codec.load_file(os.path.join(GOLDEN, f"catalog_{name}.rec.xz"))).all()
    text = open(os.path.join(GOLDEN, "configs", name + ".json")).read()
    reports, _, sampled, _ = oracle.run_detection_cfg(text, recs)
    assert fnv1a64(reports.encode()) == MANIFEST[name]["reports_fnv1a64"]
    assert sampled == MANIFEST[name]["sampled"]
