"""Sharded timeline: torchrun --nproc-per-node N scripts/timeline_multi.py;
rank 0 prints its kernel + NCCL timeline of the last (profiled) step."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank = int(os.environ["RANK"])
ws = int(os.environ["WORLD_SIZE"])
if rank == 0:
    os.environ["CSG_TIMELINE"] = "1"
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
import bench  # noqa: E402
from paper_2509_03018_b200 import distributed as D  # noqa: E402
from paper_2509_03018_b200 import engine as E  # noqa: E402

scen, recs = bench.load_workload(ws, rank)
topo, prog = scen.layout()
tcfg, acfg, seed = scen.configs()
ctx = E.Context(rank)
D.init_engine_comm(ctx)
store = E.TraceStore(ctx)
store.append(recs)
model = E.Model(topo, prog, ctx)
for i in range(4):
    store.invalidate()
    ctx.profile(i == 3)
    dist.barrier()
    E.run_detection(store, model, tcfg, acfg, seed)
    if i == 3:
        if rank == 0:
            print("---- last step", file=sys.stderr, flush=True)
        ctx.kernel_stats()

# per-rank device time per step, back to back (as bench.py) and barrier-separated
for mode in ("back-to-back", "barrier"):
    ctx.reset_stats()
    ctx.profile(False)
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(10):
        if mode == "barrier":
            dist.barrier()
        store.invalidate()
        E.run_detection(store, model, tcfg, acfg, seed)
    ms, _ = ctx.stats()
    print(f"rank {rank} {mode}: {ms / 10:.3f} ms/step", file=sys.stderr, flush=True)
dist.destroy_process_group()
