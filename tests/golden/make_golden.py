"""Regenerates the golden fixtures from the reference itself.

    python -m tests.golden.make_golden

Needs oracle/_ref (built from /root/reference by `make -C oracle`). For each
catalog scenario config (copied verbatim from the reference's
proj/configs/ as test data) the reference simulator produces the trace and
the reference run_detection + reports_to_jsonl produce the expected output:

  catalog_<name>.rec.xz       packed records (tests/golden/codec.py)
  catalog_<name>.reports.jsonl reports_to_jsonl bytes (reference)
  catalog_<name>.full.jsonl    structured reports incl. exonerated lists
  manifest.json               record counts, sampled ranks, FNV-1a-64 hashes
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from tests.golden import codec  # noqa: E402

CATALOG = ["clean"] + [f"scenario{i}" for i in range(1, 8)]


def fnv1a64(data: bytes) -> str:
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def main():
    manifest = {}
    for name in CATALOG:
        cfg = open(os.path.join(HERE, "configs", f"{name}.json")).read()
        recs = ref.simulate(cfg)
        reports, full, sampled, _ = ref.run_detection_cfg(cfg, recs)
        codec.save_file(os.path.join(HERE, f"catalog_{name}.rec.xz"), recs)
        with open(os.path.join(HERE, f"catalog_{name}.reports.jsonl"), "w") as f:
            f.write(reports)
        with open(os.path.join(HERE, f"catalog_{name}.full.jsonl"), "w") as f:
            for r in full:
                f.write(json.dumps(r) + "\n")
        manifest[name] = {"records": int(len(recs)), "sampled": sampled,
                          "outcomes": len(full),
                          "reports_fnv1a64": fnv1a64(reports.encode())}
        print(name, manifest[name])
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
