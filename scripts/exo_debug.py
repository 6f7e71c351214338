"""One detection replay of the bench store with CSG_DEBUG_EXO=1 (candidate /
op-DAG sizes per trip printed by k_exonerate) and per-kernel device times."""
import os
import sys

os.environ["CSG_DEBUG_EXO"] = "1"
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
for i in range(3):
    store.invalidate()
    if i == 2:
        ctx.reset_stats()
        ctx.profile(True)
    reps, _ = E.run_detection(store, model, tcfg, acfg, seed)
ms, launches = ctx.stats()
k, _, _ = ctx.kernel_stats()
tot = sum(v[0] for v in k.values())
print(f"step {ms:.3f} ms, kernels {tot:.3f} ms, launches {launches}")
for name, (t, n) in sorted(k.items(), key=lambda kv: -kv[1][0]):
    print(f"  {name:24s} {n:4d} {t * 1e3:9.1f} us")
print("trips", len(reps), [len(r.get("suspects", [])) for r in reps],
      [len(r.get("exonerated", [])) for r in reps])
