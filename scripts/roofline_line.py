"""One-line summary of a bench JSON line: roofline kernel, launch time, frac, step."""
import json
import sys

d = json.load(open(sys.argv[1]))
r = d["roofline"]
print(r["kernel"], round(r["avg_launch_ms"] * 1e3, 1), "us frac", round(r["frac"], 3),
      "step", round(d["ms_per_step"], 4))
