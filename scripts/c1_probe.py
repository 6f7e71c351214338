import time, json, hashlib
from oracle import ref
from paper_2509_03018_b200.model import OpProgram, CollOpSpec
cfg = open('configs/c1_ring_32.json').read()
prog = OpProgram([CollOpSpec(0, 2, 0)])
t=time.time(); recs = ref.simulate_prog(cfg, prog, 1<<27); print(len(recs), time.time()-t)
topo, _ = ref.layout(1,1,32,1,4,4)
print("last ts", recs["ts"].max(), "kinds", (recs["kind"]==0).sum())
print(topo.groups[0])
sc = json.loads(cfg)
from paper_2509_03018_b200 import engine
scen = engine.Scenario.load('configs/c1_ring_32.json')
tcfg, acfg, seed = scen.configs()
print(tcfg, acfg, seed)
rep, full, secs = ref.run_detection(topo, prog, tcfg, acfg, seed, recs, onset=30004.0)
print(secs, len(full)); print(rep[:1500])
