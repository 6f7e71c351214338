"""Host half of the trace generator (synth.cpp: op-instance schedule + the
shared flow expansion of synth_flow.h) on the CPU: the catalog synthetic
traces keep the bytes the reference-pinned fixtures were made from
(manifest.json), C1 keeps its digest, a target cut of a shard holds
exactly the target and only the shard's ranks. The device expansion is held to
these same bytes by tests/test_gpu_synth.py."""
import json
import os

import pytest

from tests.conftest import GOLDEN, ROOT
from tests.golden.make_golden import fnv1a64

MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))


@pytest.mark.parametrize("name", ["synth_hang_128", "synth_strag_128"])
def test_catalog_synth_bytes(eng, name):
    recs = eng.synthesize(eng.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json")), 0)
    assert len(recs) == MANIFEST[name]["records"]
    assert fnv1a64(recs.tobytes()) == MANIFEST[name]["records_fnv1a64"]


@pytest.mark.parametrize("cfg,target,ranks,n,digest", [
    ("configs/c1_ring_32.json", 0, None, 293191, "de74f8cb0c524840"),
    ("configs/c1_ring_32.json", 100000, (4, 20), 100000, None),
])
def test_benchmark_synth_digests(eng, cfg, target, ranks, n, digest):
    recs = eng.synthesize(eng.Scenario.load(os.path.join(ROOT, cfg)), target, ranks)
    assert len(recs) == n
    if digest:
        assert fnv1a64(recs.tobytes()) == digest
    if ranks:
        assert ((recs["rank"] >= ranks[0]) & (recs["rank"] < ranks[1])).all()


def test_shards_partition_the_trace(eng):
    """Rank-range shards of one trace are disjoint and together hold it."""
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", "synth_hang_128.json"))
    full = eng.synthesize(scen, 0)
    parts = [eng.synthesize(scen, 0, (lo, lo + 32)) for lo in range(0, 128, 32)]
    assert sum(len(p) for p in parts) == len(full)
    for lo, p in zip(range(0, 128, 32), parts):
        assert ((p["rank"] >= lo) & (p["rank"] < lo + 32)).all()


def test_copy_side_faults_take_copy_factor(eng):
    """pcie_downgrade / gpu_power_limit / background_compute slow copies in
    the reference (sim.cpp copy_factor); the generator's per-rank slowdown
    takes whichever factor the fault sets, so a copy_factor fault slows the
    rank exactly as the same bandwidth_factor one did, and differs from a
    fault-free trace."""
    cfg = json.load(open(os.path.join(GOLDEN, "configs", "synth_strag_128.json")))
    f = [x for x in cfg["faults"] if x["kind"] == "pcie_downgrade"][0]
    assert "bandwidth_factor" in f and "copy_factor" not in f

    def synth(faults):
        c = dict(cfg, faults=faults)
        return eng.synthesize(eng.Scenario.parse(json.dumps(c)), 0).tobytes()

    by_bw = synth([f])
    g = {k: v for k, v in f.items() if k != "bandwidth_factor"}
    g["copy_factor"] = f["bandwidth_factor"]
    assert synth([g]) == by_bw
    assert synth([]) != by_bw
