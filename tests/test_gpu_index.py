"""The two device index builders must produce the same rank-major store:
the fused one-pass counting sort (k_stats_hist -> k_scatter, rank spans up to
2048, sub-tiles of 2048 or 1024 records) and the general LSD radix sort +
gather (CSG_INDEX_RADIX=1, any span). The general path is itself pinned to
the reference on the catalog (test_gpu_catalog runs both). Compared here on
shapes the catalog does not reach: 1024 < span <= 2048 (wide sub-tiles), a
shard whose ranks start above 0 (rotated digits), and a ragged last tile."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, %(root)r)
from paper_2509_03018_b200 import engine as E
from paper_2509_03018_b200._abi import RECORD_DTYPE
cfg = json.load(open(os.path.join(%(root)r, 'configs', 'c2_mini_128.json')))
cfg['layout']['dp'] = %(dp)d
cfg['sim']['max_sim_ms'] = 2600.0
cfg['faults'][0]['onset_ms'] = 1504.0
scen = E.Scenario.parse(json.dumps(cfg))
recs = E.synthesize(scen, 0, (%(lo)d, %(hi)d))[: %(cut)d]
topo, prog = scen.layout()
tc, ac, seed = scen.configs()
store = E.TraceStore(records=recs)
got, sampled = E.run_detection(store, E.Model(topo, prog), tc, ac, seed)
ranks = sorted(set(np.unique(recs['rank']).tolist()))
q = [store.query(ranks[i::7], 300.0 * i, 300.0 * i + 900.0) for i in range(7)]
ll = store.last_log_per_rank(ranks[::5], 1700.0)
print(json.dumps({'n': len(recs), 'reports': got, 'q': q, 'll': ll}))
"""


def run(env_extra, **kw):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD % dict(root=ROOT, **kw)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("dp,lo,hi,cut", [
    (96, 0, 1 << 30, 10 ** 9),        # 1536 ranks: span > 1024 (1024-record sub-tiles)
    (96, 700, 1900, 10 ** 9),         # shard [700, 1900): rotated digits, rank base 700
    (64, 0, 1 << 30, 4096 * 37 + 5),  # 1024 ranks, ragged last tile
])
def test_fused_index_matches_radix_index(dp, lo, hi, cut):
    a = run({}, dp=dp, lo=lo, hi=hi, cut=cut)
    b = run({"CSG_INDEX_RADIX": "1"}, dp=dp, lo=lo, hi=hi, cut=cut)
    assert a["n"] == b["n"] and a["n"] > 0
    assert a["q"] == b["q"]
    assert a["ll"] == b["ll"]
    assert a["reports"] == b["reports"]


SPEC_CHILD = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, %(root)r)
from paper_2509_03018_b200 import engine as E
cfg = json.load(open(os.path.join(%(root)r, 'configs', 'c2_mini_128.json')))
cfg['layout']['dp'] = %(dp)d
cfg['sim']['max_sim_ms'] = 2600.0
cfg['faults'][0]['onset_ms'] = 1504.0
scen = E.Scenario.parse(json.dumps(cfg))
full = E.synthesize(scen, 0, (0, 1 << 30))
topo, prog = scen.layout()
tc, ac, seed = scen.configs()
model = E.Model(topo, prog)
store = E.TraceStore()
part = full[(full['rank'] >= 100) & (full['rank'] < 900)]
bad = full[:5000].copy()
bad['rank'][77] = -3
steps = [full, full, part, part[: len(part) * 2 // 3], full, bad, full, full]
out = []
for recs in steps:
    store.clear()
    store.append(recs)
    try:
        got, sampled = E.run_detection(store, model, tc, ac, seed)
        ranks = sorted(set(np.unique(recs['rank']).tolist()))
        q = [store.query(ranks[i::7], 300.0 * i, 300.0 * i + 900.0) for i in range(7)]
        out.append({'n': len(recs), 'reports': got, 'q': q})
    except Exception as e:
        out.append({'error': type(e).__name__})
print(json.dumps(out))
"""


@pytest.mark.gpu
@pytest.mark.parametrize("dp", [64, 160])
def test_speculative_index_layout_matches_fresh_builds(dp):
    """Rebuilding one store over the same rank layout launches the index on
    the last layout before the statistics reach the host (store_build_index);
    hits (same span, any n), misses (other span) and invalid input must give
    exactly what builds without speculation give. dp=160 (2560 ranks) takes
    the general path, whose rebuilds write the sort pairs in the statistics
    pass (and miss to the fused path for the narrow slices)."""
    def go(env_extra):
        env = dict(os.environ, **env_extra)
        r = subprocess.run([sys.executable, "-c", SPEC_CHILD % dict(root=ROOT, dp=dp)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return json.loads(r.stdout.strip().splitlines()[-1])
    a = go({})
    b = go({"CSG_INDEX_NOSPEC": "1"})
    assert len(a) == len(b) == 8
    assert a[5] == b[5] == {"error": a[5].get("error")} and "error" in a[5]
    for x, y in zip(a, b):
        assert x == y
