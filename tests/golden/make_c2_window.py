"""Regenerates tests/golden/c2_window.json: the reference analyzer's
report for one detection window (evaluate at t=22000 + analyze of its
trigger) over the full benchmark store (configs/c2_hang_1024.json, 1e7
records). Takes ~11 minutes on one core (the reference's exoneration BFS).

    python -m tests.golden.make_c2_window
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2509_03018_b200 import engine as E  # noqa: E402
from tests.golden.make_golden import fnv1a64  # noqa: E402


def main():
    cfg_path = os.path.join(ROOT, "configs", "c2_hang_1024.json")
    recs = E.synthesize(E.Scenario.load(cfg_path), 10_000_000)
    store = ref.RefStore(recs)
    t0 = time.time()
    cfg = json.load(open(cfg_path))
    onset = cfg["faults"][0]["onset_ms"]
    I = cfg["trigger"]["detect_interval_ms"]
    t = I
    while t < onset:  # first detection tick at or after the injected hang
        t += I
    e, a, tripped, rep = store.window(open(cfg_path).read(), t)
    out = {"config": "configs/c2_hang_1024.json", "target_records": 10_000_000,
           "records": int(len(recs)), "records_fnv1a64": fnv1a64(recs.tobytes()),
           "window_t": t, "reference_evaluate_s": e, "reference_analyze_s": a,
           "note": "reference evaluate + analyze at the first tripped tick over the "
                   "full C2 store (oracle/_ref, 1 core)", "report": rep}
    json.dump(out, open(os.path.join(HERE, "c2_window.json"), "w"))
    print(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
