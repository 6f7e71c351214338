"""Per-kernel CUDA-event times of one detection replay of the bench store
(3 warm steps, then 3 profiled steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_03018_b200 import engine as E  # noqa: E402

scen, recs = bench.load_workload(1, 0)
topo, prog = scen.layout()
tcfg, acfg, seed = scen.configs()
ctx = E.Context(0)
store = E.TraceStore(ctx)
store.append(recs)
model = E.Model(topo, prog, ctx)
for i in range(6):
    if i == 3:
        ctx.reset_stats()
        ctx.profile(True)
    store.invalidate()
    E.run_detection(store, model, tcfg, acfg, seed)
k, _, _ = ctx.kernel_stats()
tag = os.environ.get("TAG", "")
for name, (t, n) in sorted(k.items(), key=lambda kv: -kv[1][0])[:6]:
    print(f"{tag} {name:22s} {t / n * 1e3:8.1f} us")
