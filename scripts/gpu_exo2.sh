#!/bin/bash
# Exoneration check: GPU suite, C3 paths, C3 bench, the 4x C3 phase breakdown.
set -u
O=gpurun_out/${1:-exo2}
mkdir -p "$O"
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest_gpu $?" >> "$O/status"
timeout 500 python scripts/c3_paths.py > "$O/c3_paths.json" 2> "$O/c3_paths.err"
echo "c3_paths $? $(tail -1 $O/c3_paths.json)" >> "$O/status"
timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-jsonl > "$O/bench_c3.json" 2> "$O/bench_c3.err"
echo "bench c3 $? $(python scripts/roofline_line.py $O/bench_c3.json 2>&1 | tail -1)" >> "$O/status"
timeout 900 python scripts/exo_c3x4.py > "$O/exo_c3x4.txt" 2>&1
echo "exo x4 $?" >> "$O/status"
cat "$O/status"
