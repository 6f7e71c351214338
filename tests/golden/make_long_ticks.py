"""Golden fixtures for detection runs with more ticks than the trigger's
one-launch path holds (T > 4266: T * 48 B of per-tick bins no longer fit in
shared memory), which take the tiled window-statistics path
(k_window_bins over 4096-tick tiles -> k_ema_ticks -> k_pick_trips).

    python -m tests.golden.make_long_ticks

Catalog traces (committed by make_golden) replayed by the REFERENCE
run_detection with a fine detection interval; the expected outputs are the
FNV-1a-64 hashes of its reports_to_jsonl bytes and of the structured reports
(one JSON line each, json.dumps default separators), plus the outcome count
and the trigger list, in long_ticks.json. Takes ~1 min of reference time.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from tests.golden import codec  # noqa: E402
from tests.golden.make_golden import fnv1a64  # noqa: E402

# (catalog trace, detect_interval_ms): scenario3 is a hang (failure trips),
# scenario7 a fail-slow run (straggler trips), clean trips nowhere
CASES = [("scenario3", 2.5), ("scenario7", 5.0), ("clean", 1.0)]


def config(name: str, interval: float) -> str:
    cfg = json.load(open(os.path.join(HERE, "configs", f"{name}.json")))
    cfg["trigger"]["detect_interval_ms"] = interval
    return json.dumps(cfg)


def _canon(x):
    # numbers as repr(float): the engine returns doubles where the parsed
    # reference JSON may hold ints (2500 vs 2500.0), which compare equal
    if isinstance(x, dict):
        return {k: _canon(v) for k, v in x.items()}
    if isinstance(x, list):
        return [_canon(v) for v in x]
    if isinstance(x, (int, float)) and not isinstance(x, bool):
        return repr(float(x))
    return x


def full_hash(full) -> str:
    return fnv1a64("".join(json.dumps(_canon(r)) + "\n" for r in full).encode())


def main():
    out = {}
    for name, interval in CASES:
        cfg = config(name, interval)
        recs = codec.load_file(os.path.join(HERE, f"catalog_{name}.rec.xz"))
        reports, full, sampled, secs = ref.run_detection_cfg(cfg, recs)
        out[f"{name}@{interval}"] = {
            "trace": name, "detect_interval_ms": interval,
            "outcomes": len(full), "sampled": sampled,
            "triggers": [[r["kind"], r["suspect_rank"], r["time_ms"]] for r in full],
            "reports_fnv1a64": fnv1a64(reports.encode()),
            "full_fnv1a64": full_hash(full),
            "reference_seconds": round(secs, 1)}
        print(name, interval, len(full), f"{secs:.1f}s", flush=True)
    with open(os.path.join(HERE, "long_ticks.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
