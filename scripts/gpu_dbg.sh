#!/bin/bash
# Phase breakdowns: k_exonerate on C3 (CSG_DEBUG_EXO), k_scatter on C2
# (CSG_DEBUG_SCATTER).
set -u
O=gpurun_out/${1:-dbg}
mkdir -p "$O"
CSG_DEBUG_EXO=1 timeout 300 python -c "
import sys
import bench
from paper_2509_03018_b200 import engine as E
bench.select_workload('c3')
scen, recs = bench.load_workload(1, 0)
t, p = scen.layout(); tc, ac, seed = scen.configs()
s = E.TraceStore(records=recs); m = E.Model(t, p)
E.run_detection(s, m, tc, ac, seed)
" > "$O/exo_debug.txt" 2>&1
echo "exo debug $?" >> "$O/status"
CSG_DEBUG_SCATTER=1 timeout 300 python scripts/kbench.py > "$O/scatter_debug.txt" 2>&1
echo "scatter debug $?" >> "$O/status"
cat "$O/status"
timeout 420 python -m pytest tests/test_gpu_selfev.py -x -q > "$O/pytest_selfev.log" 2>&1
echo "pytest selfev $?" >> "$O/status"
CSG_DEBUG_SF=1 timeout 500 python scripts/c3_paths.py > "$O/c3_paths.json" 2> "$O/c3_paths.err"
echo "c3_paths $? $(cat $O/c3_paths.json | tail -1)" >> "$O/status"
timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-jsonl > "$O/bench_c3.json" 2> "$O/bench_c3.err"
echo "bench c3 $? $(python scripts/roofline_line.py "$O/bench_c3.json" 2>&1 | tail -1)" >> "$O/status"
cat "$O/status"
