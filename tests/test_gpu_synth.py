"""The device trace generator (synth_gpu.cu: host-scheduled flows expanded,
ordered and appended on the GPU) must produce exactly the host generator's
bytes (host/synth.cpp), whose catalog outputs are pinned to the reference
analyzer (test_gpu_catalog, manifest.json)."""
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

CASES = [
    (os.path.join(GOLDEN, "configs", "synth_hang_128.json"), 0, None),
    (os.path.join(GOLDEN, "configs", "synth_strag_128.json"), 0, None),
    (os.path.join(ROOT, "configs", "c2_hang_1024.json"), 3_000_000, None),  # target cut
    (os.path.join(ROOT, "configs", "c2_hang_1024.json"), 0, (100, 700)),    # one shard
    (os.path.join(ROOT, "configs", "c3_mini_1024.json"), 0, None),          # fail-slow
    (os.path.join(ROOT, "configs", "c1_ring_32.json"), 0, None),
]


@pytest.mark.parametrize("cfg,target,ranks", CASES)
def test_device_generator_matches_host(eng, cfg, target, ranks):
    scen = eng.Scenario.load(cfg)
    want = eng.synthesize(scen, target, ranks)
    store = eng.TraceStore()
    n = eng.synthesize_into(store, scen, target, ranks)
    assert n == len(want)
    got = store.records()
    assert got.dtype == want.dtype
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


def test_device_generator_appends(eng):
    """Appends after records already in the store (a shard built in parts)."""
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", "synth_hang_128.json"))
    a = eng.synthesize(scen, 0, (0, 64))
    b = eng.synthesize(scen, 0, (64, 128))
    store = eng.TraceStore(records=a)
    assert eng.synthesize_into(store, scen, 0, (64, 128)) == len(b)
    got = store.records()
    # raw bytes: concatenating the union-layout record dtype would repack it
    want = np.concatenate([a.view(np.uint8), b.view(np.uint8)])
    assert np.array_equal(got.view(np.uint8), want)
