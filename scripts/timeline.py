"""One detection replay of the bench store with CSG_TIMELINE=1: every
kernel's start, duration and the idle gap before it (host round trips)."""
import os
import sys

os.environ["CSG_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_03018_b200 import engine as E  # noqa: E402

if len(sys.argv) > 1:  # python scripts/timeline.py c3
    bench.select_workload(sys.argv[1])

scen, recs = bench.load_workload(1, 0)
topo, prog = scen.layout()
tcfg, acfg, seed = scen.configs()
ctx = E.Context(0)
store = E.TraceStore(ctx)
store.append(recs)
model = E.Model(topo, prog, ctx)
for i in range(4):
    store.invalidate()
    ctx.profile(i == 3)
    reps, _ = E.run_detection(store, model, tcfg, acfg, seed)
    if i == 3:
        print("---- last step", file=sys.stderr)
        ctx.kernel_stats()
