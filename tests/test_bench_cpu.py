"""bench.py workload plumbing (host only): weak-scaling jobs grow DP with N,
the fixed C4 job keeps its 65,536-rank layout and shards it by rank range."""
import json

import bench
from paper_2509_03018_b200 import distributed as D


def _layout(n):
    return json.loads(bench.scaled_config(n))["layout"]


def test_c2_weak_scaling_grows_dp():
    bench.select_workload("c2")
    for n in (1, 2, 4, 8):
        lay = _layout(n)
        assert lay["dp"] == 32 * n
        assert lay["tp"] * lay["pp"] * lay["dp"] == 1024 * n


def test_c4_is_a_fixed_job():
    try:
        bench.select_workload("c4")
        for n in (1, 2, 4, 8):
            lay = _layout(n)
            world = lay["tp"] * lay["pp"] * lay["dp"]
            assert world == 65536
            b = D.shard_bounds(world, n)
            assert b[0][0] == 0 and len(b) == n
            assert all(b[i][1] == b[i + 1][0] for i in range(n - 1))
            if n > 1:
                assert b[-2][1] == world * (n - 1) // n
        assert "c4" in bench.FIXED_JOB
    finally:
        bench.select_workload("c2")
