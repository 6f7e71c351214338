"""One profiled detection replay of a bench workload with the timeline:
    python scripts/probe_workload.py c3"""
import os
import sys
import time

os.environ["CSG_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_03018_b200 import engine as E  # noqa: E402

bench.select_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
scen, recs = bench.load_workload(1, 0)
topo, prog = scen.layout()
tcfg, acfg, seed = scen.configs()
ctx = E.Context(0)
store = E.TraceStore(ctx)
store.append(recs)
model = E.Model(topo, prog, ctx)
ctx.profile(True)
t = time.time()
reps, sampled = E.run_detection(store, model, tcfg, acfg, seed)
print(f"replay {time.time() - t:.2f} s, {len(reps)} trips, kinds",
      sorted({r.get("kind", r.get("trigger_kind")) for r in reps}) if reps else [], file=sys.stderr)
print("---- last step", file=sys.stderr)
ctx.kernel_stats()
