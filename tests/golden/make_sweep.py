"""Regenerates the C5 fault-injection sweep fixtures
from the reference itself.

    python -m tests.golden.make_sweep

Base layout: the reference catalog's (tp 8, pp 2, dp 2, 8 ranks per node,
2 channels per pair, 4 NICs; proj/configs/). Each case is either a reference
simulator fault (run_simulation, proj/src/sim.cpp) or a deterministic
record-level edit of a reference-simulated trace; the expected reports are the
reference run_detection + reports_to_jsonl over the final records
(proj/src/runner.cpp:47-169):

  sweep_gpu_down     a silenced node: nic_shutdown on all 4 NICs of node 2,
                     logs stop 500 ms after onset
  sweep_nic_flap     clean trace with node 1's channel-0 records dropped over
                     [3000, 3600] ms (NIC down, then recovery)
  sweep_slow_pcie    pcie_downgrade on rank 9, copy_factor 0.05
  sweep_opseq_lag    the scenario-1 hang with ranks 1 and 20 logging op_seq
                     one behind from 2000 ms on (exercises check_min_op)

Writes catalog_<case>.rec.xz / .reports.jsonl / .full.jsonl, configs/<case>.json
and the manifest entries (so tests/test_gpu_catalog.py's golden() loads them).
"""
from __future__ import annotations

import copy
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from tests.golden import codec  # noqa: E402
from tests.golden.make_golden import fnv1a64  # noqa: E402

CASES = ["sweep_gpu_down", "sweep_nic_flap", "sweep_slow_pcie", "sweep_opseq_lag"]


def _base():
    return json.load(open(os.path.join(HERE, "configs", "scenario1.json")))


def case(name):
    """-> (config dict, packed records)"""
    cfg = _base()
    if name == "sweep_gpu_down":
        cfg["faults"] = [{"kind": "nic_shutdown", "node": 2, "nic": k,
                          "onset_ms": 3004.0, "stop_logs_after_ms": 500.0}
                         for k in range(4)]
        return cfg, ref.simulate(json.dumps(cfg))
    if name == "sweep_slow_pcie":
        cfg["faults"] = [{"kind": "pcie_downgrade", "rank": 9, "onset_ms": 2504.0,
                          "copy_factor": 0.05}]
        return cfg, ref.simulate(json.dumps(cfg))
    if name == "sweep_nic_flap":
        clean = copy.deepcopy(cfg)
        clean["faults"] = []
        recs = ref.simulate(json.dumps(clean))
        node1 = (recs["rank"] >= 8) & (recs["rank"] < 16)
        gap = node1 & (recs["channel"] == 0) & (recs["ts"] >= 3000.0) & \
            (recs["ts"] <= 3600.0)
        cfg["faults"] = [{"kind": "nic_shutdown", "node": 1, "nic": 0,
                          "onset_ms": 3000.0}]  # onset for latency_ms only
        return cfg, recs[~gap].copy()
    if name == "sweep_opseq_lag":
        recs = ref.simulate(json.dumps(cfg))
        lag = np.isin(recs["rank"], [1, 20]) & (recs["ts"] >= 2000.0) & \
            (recs["op_seq"] > 0)
        recs = recs.copy()
        recs["op_seq"][lag] -= 1
        return cfg, recs
    raise KeyError(name)


def main():
    path = os.path.join(HERE, "manifest.json")
    manifest = json.load(open(path))
    for name in CASES:
        cfg, recs = case(name)
        text = json.dumps(cfg, indent=1)
        with open(os.path.join(HERE, "configs", name + ".json"), "w") as f:
            f.write(text + "\n")
        reports, full, sampled, _ = ref.run_detection_cfg(text, recs)
        codec.save_file(os.path.join(HERE, f"catalog_{name}.rec.xz"), recs)
        with open(os.path.join(HERE, f"catalog_{name}.reports.jsonl"), "w") as f:
            f.write(reports)
        with open(os.path.join(HERE, f"catalog_{name}.full.jsonl"), "w") as f:
            for r in full:
                f.write(json.dumps(r) + "\n")
        manifest[name] = {"records": int(len(recs)), "sampled": sampled,
                          "outcomes": len(full),
                          "records_fnv1a64": fnv1a64(recs.tobytes()),
                          "reports_fnv1a64": fnv1a64(reports.encode())}
        print(name, len(recs), len(full), sorted({r["verdict"] for r in full}),
              sorted({r["kind"] for r in full}))
    with open(path, "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
