"""Sharded (multi-GPU) parity: records split by rank range over 2+ GPUs,
combined by the engine's NCCL collectives, must give the single-store
reference reports exactly, on every rank. Skipped on a 1-GPU box."""
import json
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from tests.conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

CASES = ["scenario1", "scenario3", "scenario7", "synth_hang_128", "synth_strag_128",
         "sweep_gpu_down", "sweep_slow_pcie", "sweep_opseq_lag"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2509_03018_b200 import distributed as D
        from paper_2509_03018_b200 import engine as E
        from tests.test_gpu_catalog import golden
        ctx = E.Context(rank)
        D.init_engine_comm(ctx)
        res = {}
        for name in CASES:
            recs, _, full = golden(name)
            scen = E.Scenario.load(os.path.join(GOLDEN, "configs", name + ".json"))
            topo, prog = scen.layout()
            tc, ac, seed = scen.configs()
            shard = D.shard_records(recs, topo.world_size, world, rank)
            store = E.TraceStore(ctx, shard)
            got, _ = E.run_detection(store, E.Model(topo, prog, ctx), tc, ac, seed)
            res[name] = got == full
        # C1: the 32-rank ring AllReduce program (tests/test_c1.py)
        from tests.test_c1 import VARIANTS, golden as c1_golden, layout as c1_layout
        topo, prog, _ = c1_layout()
        for name in VARIANTS:
            recs, full = c1_golden(name)
            cfg = open(os.path.join(GOLDEN, "configs", name + ".json")).read()
            tc, ac, seed = E.Scenario.parse(cfg).configs()
            shard = D.shard_records(recs, topo.world_size, world, rank)
            store = E.TraceStore(ctx, shard)
            got, _ = E.run_detection(store, E.Model(topo, prog, ctx), tc, ac, seed)
            res[name] = got == full
        q.put((rank, res, ctx.comm_info()))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_sharded_matches_reference():
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, res, info in out:
        assert all(res.values()), (rank, res)
        assert info[0] == world and info[2] > 0  # collectives were issued
