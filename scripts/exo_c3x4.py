"""k_exonerate phase breakdown on the C3 shape at 4x the ranks (the job the
4-GPU weak-scaling C3 line analyzes), on one GPU: CSG_DEBUG_EXO=1 output,
largest trips first."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys
sys.path.insert(0, %(root)r)
from paper_2509_03018_b200 import engine as E
cfg = json.load(open(%(root)r + '/configs/c3_8192.json'))
cfg['layout']['dp'] *= 4
s = E.Scenario.parse(json.dumps(cfg))
st = E.TraceStore()
n = E.synthesize_into(st, s, 400_000_000)
t, p = s.layout(); tc, ac, seed = s.configs()
got, _ = E.run_detection(st, E.Model(t, p), tc, ac, seed)
print('records', n, 'reports', len(got), file=sys.stderr)
"""
env = dict(os.environ, CSG_DEBUG_EXO="1")
r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}], env=env, capture_output=True,
                   text=True, timeout=900)
rows = [l for l in r.stdout.splitlines() + r.stderr.splitlines() if "exo trip" in l]
rows.sort(key=lambda l: -int(re.search(r"C=(\d+)", l).group(1)))
print("\n".join(rows[:8]))
print(r.stderr[-500:])
