"""BASELINE configs[4]: the fault-injection sweep (GPU down, NIC flap, slow
PCIe, mismatched op_seq) at the C2 scale (1024 ranks per GPU, ~1e7 records
per GPU, weak scaling like bench.py), on N GPUs, beside the reference
analyzer on the host (N = 1: one detection window per case, time-capped).

    python scripts/sweep_c5.py [--steps K]
    torchrun --nproc-per-node N scripts/sweep_c5.py

The cases follow tests/golden/make_sweep.py (which pins them to the
reference at the catalog scale), scaled to the C2 layout: all NICs of a node
shut with logs stopping (GPU down), all of a sampled node's records dropped
for 600 ms then back (NIC flap), pcie_downgrade on one rank (slow PCIe), two
ranks logging op_seq one behind after the C2 hang's onset (mismatched
op_seq). Prints one JSON line (rank 0)."""
import argparse
import copy
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cases(base, victim):
    """victim: a rank the trigger samples (the faults of this sweep are local,
    so a flap or a slow PCIe link far from every sampled rank never trips)."""
    node = victim // base["layout"]["ranks_per_node"]
    out = {}
    c = copy.deepcopy(base)
    c["faults"] = [{"kind": "nic_shutdown", "node": 37, "nic": k, "onset_ms": 22004.0,
                    "stop_logs_after_ms": 1000.0} for k in range(4)]
    out["gpu_down"] = (c, c, None)
    c = copy.deepcopy(base)
    c["faults"] = [{"kind": "pcie_downgrade", "rank": victim, "onset_ms": 12004.0,
                    "copy_factor": 0.05}]
    out["slow_pcie"] = (c, c, None)
    clean = copy.deepcopy(base)
    clean["faults"] = []
    c = copy.deepcopy(base)
    c["faults"] = [{"kind": "nic_shutdown", "node": node, "nic": 0, "onset_ms": 15000.0}]
    rpn = base["layout"]["ranks_per_node"]

    def flap(r):
        on = (r["rank"] >= node * rpn) & (r["rank"] < (node + 1) * rpn)
        gap = on & (r["ts"] >= 15000.0) & (r["ts"] <= 15600.0)
        return r[~gap].copy()
    out["nic_flap"] = (clean, c, flap)

    def lag(r):
        m = np.isin(r["rank"], [1, 500]) & (r["ts"] >= 20000.0) & (r["op_seq"] > 0)
        r = r.copy()
        r["op_seq"][m] -= 1
        return r
    out["opseq_lag"] = (base, base, lag)
    return out


def capped_replay(cfg_text, recs, cap_s):
    """The reference's whole run_detection over the trace in a forked child,
    killed after cap_s. -> (seconds, finished, full reports or None)"""
    import multiprocessing as mp
    from oracle import ref
    ctx = mp.get_context("fork")
    q = ctx.Queue()

    def child():
        _, full, _, secs = ref.run_detection_cfg(cfg_text, recs)
        q.put((secs, full))

    p = ctx.Process(target=child)
    t0 = time.perf_counter()
    p.start()
    try:
        secs, full = q.get(timeout=cap_s)
    except Exception:
        p.kill()
        p.join()
        return time.perf_counter() - t0, False, None
    p.join()
    return secs, True, full


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-cap", type=float, default=45.0)
    ap.add_argument("--cpu-replay", default="slow_pcie,nic_flap",
                    help="cases whose whole detection replay also runs on the "
                         "reference analyzer (N = 1), reports compared")
    ap.add_argument("--replay-cap", type=float, default=300.0)
    ap.add_argument("--cases", default="", help="comma list (default: all)")
    ap.add_argument("--timeline", default="",
                    help="case whose last replay rank 0 prints as a kernel/NCCL timeline")
    args = ap.parse_args()
    if args.timeline and int(os.environ.get("RANK", "0")) == 0:
        os.environ["CSG_TIMELINE"] = "1"
    import torch
    import torch.distributed as dist
    import bench
    from paper_2509_03018_b200 import distributed as D
    from paper_2509_03018_b200 import engine as E
    ws, rank, local = bench.dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base = json.load(open(os.path.join(ROOT, "configs", "c2_hang_1024.json")))
    base["layout"]["dp"] *= ws
    base["sim"]["max_sim_ms"] = 26000.0
    world = base["layout"]["tp"] * base["layout"]["pp"] * base["layout"]["dp"]
    lo, hi = D.shard_bounds(world, ws)[rank]
    ctx = E.Context(local)
    if ws > 1:
        D.init_engine_comm(ctx)
    scen0 = E.Scenario.parse(json.dumps(base))
    t0, p0 = scen0.layout()
    tc0, _, seed0 = scen0.configs()
    m0 = E.Model(t0, p0, ctx)
    victim = E.sample_ranks(m0, tc0.max_sampled_ranks, seed0)[0]
    m0.close()
    res = {}
    for name, (trace_cfg, cfg, edit) in cases(base, victim).items():
        if args.cases and name not in args.cases.split(","):
            continue
        recs = bench.synthesize(E, E.Scenario.parse(json.dumps(trace_cfg)), 0,
                                (lo, hi) if ws > 1 else None)
        if edit:
            recs = edit(recs)
        scen = E.Scenario.parse(json.dumps(cfg))
        topo, prog = scen.layout()
        tcfg, acfg, seed = scen.configs()
        store = E.TraceStore(ctx)
        store.append(recs)
        model = E.Model(topo, prog, ctx)
        for _ in range(args.warmup):
            store.invalidate()
            out = E.run_detection_results(store, model, tcfg, acfg, seed)
        ctx.reset_stats()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        for _ in range(args.steps):
            if ws > 1:
                dist.barrier()
            store.invalidate()
            out = E.run_detection_results(store, model, tcfg, acfg, seed)
        ms, _ = ctx.stats()
        ms /= args.steps
        if name == args.timeline:
            ctx.profile(True)
            if ws > 1:
                dist.barrier()
            store.invalidate()
            E.run_detection_results(store, model, tcfg, acfg, seed)
            if rank == 0:
                print("---- timeline", name, file=sys.stderr, flush=True)
            ctx.kernel_stats()
            ctx.profile(False)
        n = len(recs)
        if ws > 1:
            t = torch.tensor([ms, float(n)], device="cuda", dtype=torch.float64)
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
            ms, n = float(t[0].item()), int(t[1].item())
        reports = out[0].reports()
        r = {"records": n, "ms_per_replay": ms, "records_per_s": n / (ms / 1e3),
             "trips": len(reports),
             "verdicts": sorted({int(x["verdict"]) for x in reports})}
        if ws == 1 and reports:
            # One detection window at the first tripped tick, fresh trigger
            # state, on both sides: the GPU engine (evaluate + analyze) and the
            # reference analyzer on the host must return the same report.
            t = reports[0]["time_ms"]
            sampled = E.sample_ranks(model, tcfg.max_sampled_ranks, seed)
            trig = E.evaluate(store, sampled, t, E.TriggerState(ctx), tcfg)
            gw = E.analyze(store, model, acfg, trig) if trig is not None else None
            r["window"] = {"tick_ms": t, "gpu_tripped": gw is not None}
            from oracle import ref
            if ref.available():
                rs = ref.RefStore(recs)
                secs, fin, rep = bench._capped_windows(rs, json.dumps(cfg), [t],
                                                       args.cpu_cap)[0]
                r["cpu_reference_window"] = {
                    "seconds": secs, "finished": fin, "records_per_s": n / secs,
                    "matches_gpu_window": (rep == gw) if fin else None,
                    "cores": 1, "cap_s": args.cpu_cap}
                if name in args.cpu_replay.split(","):
                    secs, fin, full = capped_replay(json.dumps(cfg), recs, args.replay_cap)
                    r["cpu_reference_replay"] = {
                        "seconds": secs, "finished": fin,
                        "records_per_s": n / secs if fin else None,
                        "reports_identical": (full == reports) if fin else None,
                        "cpu_trips": len(full) if fin else None,
                        "cores": 1, "cap_s": args.replay_cap}
        res[name] = r
        store.close()
        model.close()
    tot_n = sum(v["records"] for v in res.values())
    tot_ms = sum(v["ms_per_replay"] for v in res.values())
    if rank == 0:
        print(json.dumps({"metric": "trace records/s through trigger+RCA (C5 fault sweep)",
                          "value": tot_n / (tot_ms / 1e3), "unit": "records/s",
                          "n_gpus": ws, "scaling": "weak", "cases": res,
                          "victim_rank": victim,
                          "data": "synthetic (device generator), C2 layout x N"}))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
