"""Debug driver for the sharded path: torchrun --nproc-per-node N scripts/multi_debug.py"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def log(*a):
    print(f"[rank {os.environ.get('RANK')} {time.strftime('%X')}]", *a, flush=True)


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    log("pg up")
    from paper_2509_03018_b200 import distributed as D
    from paper_2509_03018_b200 import engine as E
    from tests.conftest import GOLDEN
    from tests.test_gpu_catalog import golden
    ctx = E.Context(rank)
    D.init_engine_comm(ctx)
    log("engine comm up", ctx.comm_info())
    for name in sys.argv[1:] or ["scenario1"]:
        recs, _, full = golden(name)
        scen = E.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
        topo, prog = scen.layout()
        tc, ac, seed = scen.configs()
        shard = D.shard_records(recs, topo.world_size, world, rank)
        log(name, "shard records", len(shard))
        store = E.TraceStore(ctx, shard)
        store.build_index()
        log(name, "index built")
        got, _ = E.run_detection(store, E.Model(topo, prog, ctx), tc, ac, seed)
        log(name, "match", got == full, len(got), len(full), ctx.comm_info())
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
