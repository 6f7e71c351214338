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
         "sweep_gpu_down", "sweep_nic_flap", "sweep_slow_pcie", "sweep_opseq_lag"]


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
        # csg_evaluate on a sharded store: every shard returns the
        # single-store answer (windows are combined across shards)
        from oracle import ref as R
        recs, _, full = golden("scenario1")
        scen = E.Scenario.load(os.path.join(GOLDEN, "configs", "scenario1.json"))
        topo, prog = scen.layout()
        tc, ac, seed = scen.configs()
        store = E.TraceStore(ctx, D.shard_records(recs, topo.world_size, world, rank))
        model = E.Model(topo, prog, ctx)
        sampled = E.sample_ranks(model, tc.max_sampled_ranks, seed)
        st_g = E.TriggerState(ctx)
        ok = True
        if R.available():
            st_r = R.TriggerState()
            for k in range(1, 25):
                t = 500.0 * k
                ok &= E.evaluate(store, sampled, t, st_g, tc) == \
                    R.evaluate(recs, sampled, t, st_r, tc)
        res["evaluate_sharded"] = ok
        # records_scanned of affected_groups counts every shard's records
        trig = E.TriggerEvent(full[0]["kind"], full[0]["suspect_rank"], full[0]["time_ms"])
        aff, scanned = E.affected_groups(store, model, ac, trig)
        res["affected_groups"] = aff == full[0]["affected_groups"] and scanned == len(recs)
        # overlapping rank ranges (ranks interleaved over shards) are refused
        inter = recs[recs["rank"] % world == rank]
        try:
            E.run_detection(E.TraceStore(ctx, inter), model, tc, ac, seed)
            res["overlap_refused"] = False
        except E.EngineError as e:
            res["overlap_refused"] = "overlap" in str(e)
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


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_contexts_on_two_devices_one_process(eng):
    """Kernels that opt into > 48 KB of dynamic shared memory (k_scatter,
    k_trigger with > 1024 ticks, k_flow_fix) launch on a second device of the
    same process: the opt-in is per device."""
    from tests.test_gpu_catalog import golden
    recs, _, full = golden("scenario3")
    scen = eng.Scenario.load(os.path.join(GOLDEN, "configs", "scenario3.json"))
    topo, prog = scen.layout()
    tc, ac, seed = scen.configs()
    tc.detect_interval_ms = 5.0  # 2400 ticks: 115 KB of trigger bins
    out = []
    for dev in (0, 1):
        ctx = eng.Context(dev)
        store = eng.TraceStore(ctx, recs)
        got, _ = eng.run_detection(store, eng.Model(topo, prog, ctx), tc, ac, seed)
        out.append(got)
        tc2, _, _ = scen.configs()
        got2, _ = eng.run_detection(store, eng.Model(topo, prog, ctx), tc2, ac, seed)
        assert got2 == full
    assert out[0] == out[1] and len(out[0]) > 0
