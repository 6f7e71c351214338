"""C3 (8192 ranks, 16 channels, fail-slow) reports through the default
straggler paths vs the serial / per-candidate ones (CSG_SF_SLOW,
CSG_SL_SERIAL, CSG_ITER_PER_TRIP, CSG_FLOW_SCAN): prints both digests and
whether they are identical.
    python scripts/c3_paths.py [config]"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "configs", "c3_8192.json")
CHILD = r"""
import json, sys, time
sys.path.insert(0, %(root)r)
from paper_2509_03018_b200 import engine as E
s = E.Scenario.load(%(cfg)r)
recs = E.synthesize(s, 100_000_000)
t, p = s.layout(); tc, ac, seed = s.configs()
store = E.TraceStore(records=recs)
m = E.Model(t, p)
got, _ = E.run_detection(store, m, tc, ac, seed)
store.invalidate()
t0 = time.time(); got2, _ = E.run_detection(store, m, tc, ac, seed); dt = time.time() - t0
assert got == got2
print(json.dumps({"reports": got, "wall_s": dt}))
"""
KNOBS = ["CSG_SF_SLOW", "CSG_SL_SERIAL", "CSG_ITER_PER_TRIP", "CSG_FLOW_SCAN", "CSG_EXO_WARP_SWEEP",
         "CSG_COH_NO_COMPACT"]


def run(slow):
    env = {k: v for k, v in os.environ.items() if k not in KNOBS}
    if slow:
        env.update({k: "1" for k in KNOBS})
    r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT, "cfg": CFG}], env=env,
                       capture_output=True, text=True, cwd=ROOT, timeout=420)
    if r.returncode:
        print(r.stderr[-3000:])
        sys.exit(1)
    sys.stderr.write(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


a, b = run(False), run(True)
da = hashlib.sha256(json.dumps(a["reports"]).encode()).hexdigest()[:16]
db = hashlib.sha256(json.dumps(b["reports"]).encode()).hexdigest()[:16]
strag = [r for r in a["reports"] if r["kind"] == 1]
print(json.dumps({"reports": len(a["reports"]), "straggler_trips": len(strag),
                  "suspects": sum(len(r["suspects"]) for r in strag),
                  "exonerated": sum(len(r["exonerated"]) for r in strag),
                  "default_digest": da, "slow_digest": db, "identical": a["reports"] == b["reports"],
                  "default_wall_s": a["wall_s"], "slow_wall_s": b["wall_s"]}))
