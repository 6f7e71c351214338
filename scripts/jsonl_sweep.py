"""JSONL-file e2e (collsight_run_analyze on a trace file) at the C2 shape,
swept over the number of reader threads, phases on stderr (CSG_E2E_PROF).

    python scripts/jsonl_sweep.py [readers ...]
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if os.environ.get("_JSONL_CHILD"):
    from paper_2509_03018_b200 import engine as E
    scen = E.Scenario.load(sys.argv[1])
    path = sys.argv[2]
    E.run_analyze(scen, path)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        res = E.run_analyze(scen, path)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"readers": os.environ.get("CSG_JSONL_READERS"),
                      "ms": [round(t * 1e3, 2) for t in ts],
                      "triggers": int(res.trigger_count)}), flush=True)
    sys.exit(0)

import bench  # noqa: E402
from paper_2509_03018_b200 import engine as E  # noqa: E402

bench.select_workload("c2")
scen, recs = bench.load_workload()[:2]
rpn = json.load(open(bench.CONFIG))["layout"]["ranks_per_node"]
path = f"/tmp/collsight_c2_{len(recs)}.jsonl"
if not os.path.exists(path):
    E.write_trace(recs, path, rpn)
cfg_path = "/tmp/collsight_c2_scenario.json"
open(cfg_path, "w").write(bench.scaled_config(1))
print(f"{len(recs)} records, {os.path.getsize(path)} bytes", flush=True)
for r in sys.argv[1:] or ["4", "8", "14"]:
    env = dict(os.environ, _JSONL_CHILD="1", CSG_JSONL_READERS=r, CSG_E2E_PROF="1")
    subprocess.run([sys.executable, __file__, cfg_path, path], env=env, check=True)
