#!/bin/bash
# PDL A/B (CSG_NO_PDL=1) on the C2 bench line + the GPU suite.
set -u
O=gpurun_out/${1:-pdl}
mkdir -p "$O"
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest_gpu $?" >> "$O/status"
for i in 1 2; do
  for V in 0 1; do
    if [ $V = 1 ]; then export CSG_NO_PDL=1; else unset CSG_NO_PDL; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-jsonl > "$O/bench_nopdl$V.$i.json" 2> "$O/bench_nopdl$V.$i.err"
    echo "bench nopdl=$V $? $(python scripts/roofline_line.py "$O/bench_nopdl$V.$i.json" 2>&1 | tail -1)" >> "$O/status"
  done
done
unset CSG_NO_PDL
cat "$O/status"
