"""Regenerates the C1 golden fixtures from the reference itself.

    python -m tests.golden.make_c1

SURVEY.md §8(d) C1: build_layout(tp 1, pp 1, dp 32, ranks_per_node 1,
4 channels, 4 NICs) — one 32-rank ring (comm 0) plus 64 singleton groups —
running a custom one-op program {AllReduce on comm 0, 128 MiB} for 1000
iterations with 1 MiB chunks, so all four channels carry data. A custom
program is expressible only through the C++ API, so the trace comes from the
reference run_simulation (oracle/ref_shim.cpp ref_simulate_prog) and the
expected reports from the reference run_detection (proj/src/runner.cpp:47-81)
over that program. Variants (same layout/program, the fault changes):

  c1_ring_32      nic_bandwidth_limit node 5 / NIC 1, factor 0.1 (the BASELINE
                  config: straggler triggers, verdict no_straggler)
  c1_ring_32_f001 the same NIC at factor 0.01 (exercises the suspect path)
  c1_ring_32_hang nic_shutdown node 5 / NIC 1 + stop_logs_after_ms (failure RCA)

Writes c1_<variant>.rec.xz, .reports.jsonl, .full.jsonl and adds the entries
to manifest.json.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2509_03018_b200.model import CollOpSpec, OpProgram  # noqa: E402
from tests.golden import codec  # noqa: E402
from tests.golden.make_golden import fnv1a64  # noqa: E402

ALLREDUCE = 2  # OpName::AllReduce (proj/include/collsight/types.hpp)
MSG_BYTES = 128 << 20
LAYOUT = (1, 1, 32, 1, 4, 4)  # tp, pp, dp, ranks_per_node, channels, nics
FAULTS = {
    "c1_ring_32": {"kind": "nic_bandwidth_limit", "node": 5, "nic": 1,
                   "onset_ms": 30004.0, "bandwidth_factor": 0.1},
    "c1_ring_32_f001": {"kind": "nic_bandwidth_limit", "node": 5, "nic": 1,
                        "onset_ms": 30004.0, "bandwidth_factor": 0.01},
    "c1_ring_32_hang": {"kind": "nic_shutdown", "node": 5, "nic": 1,
                        "onset_ms": 30004.0, "stop_logs_after_ms": 1000.0},
}


def program() -> OpProgram:
    return OpProgram([CollOpSpec(0, ALLREDUCE, 0)])


def config_text(name: str) -> str:
    base = json.load(open(os.path.join(ROOT, "configs", "c1_ring_32.json")))
    base["faults"] = [FAULTS[name]]
    return json.dumps(base)


def main():
    path = os.path.join(HERE, "manifest.json")
    manifest = json.load(open(path))
    topo, _ = ref.layout(*LAYOUT)
    for name in FAULTS:
        cfg = config_text(name)
        with open(os.path.join(HERE, "configs", name + ".json"), "w") as f:
            f.write(cfg + "\n")
        recs = ref.simulate_prog(cfg, program(), MSG_BYTES)
        from paper_2509_03018_b200 import engine
        tcfg, acfg, seed = engine.Scenario.parse(cfg).configs()
        reports, full, _ = ref.run_detection(topo, program(), tcfg, acfg, seed,
                                             recs, onset=FAULTS[name]["onset_ms"])
        codec.save_file(os.path.join(HERE, f"{name}.rec.xz"), recs)
        with open(os.path.join(HERE, f"{name}.reports.jsonl"), "w") as f:
            f.write(reports)
        with open(os.path.join(HERE, f"{name}.full.jsonl"), "w") as f:
            for r in full:
                f.write(json.dumps(r) + "\n")
        manifest[name] = {"records": int(len(recs)), "outcomes": len(full),
                          "records_fnv1a64": fnv1a64(recs.tobytes()),
                          "reports_fnv1a64": fnv1a64(reports.encode())}
        print(name, len(recs), len(full),
              sorted({r["verdict"] for r in full}))
    with open(path, "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
