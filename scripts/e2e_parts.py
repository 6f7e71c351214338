"""Where the end-to-end C-API time goes: H2D of the packed store, the
detection replay, report rendering (bench C2 store, pinned host buffer)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_03018_b200 import engine as E  # noqa: E402

scen, recs = bench.load_workload(1, 0)
n = len(recs)
pinned = torch.empty(n * 48, dtype=torch.uint8, pin_memory=True)
host = pinned.numpy().view(recs.dtype)
host[:] = recs
topo, prog = scen.layout()
tcfg, acfg, seed = scen.configs()
ctx = E.Context(0)
store = E.TraceStore(ctx)
model = E.Model(topo, prog, ctx)
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    store.clear()
    store.append(host)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    reps, _ = E.run_detection(store, model, tcfg, acfg, seed)
    t2 = time.perf_counter()
    res = E.run_analyze_packed(scen, host)
    t3 = time.perf_counter()
    print(f"append(H2D) {1e3 * (t1 - t0):.2f} ms ({n * 48 / (t1 - t0) / 1e9:.1f} GB/s), "
          f"run_detection {1e3 * (t2 - t1):.2f} ms, full C API {1e3 * (t3 - t2):.2f} ms",
          flush=True)
