#!/bin/bash
# GPU suite + C2 and C3 bench lines.
set -u
O=gpurun_out/${1:-quick}
mkdir -p "$O"
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest_gpu $?" >> "$O/status"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > "$O/bench.json" 2> "$O/bench.err"
echo "bench c2 $? $(python scripts/roofline_line.py "$O/bench.json" 2>&1 | tail -1)" >> "$O/status"
timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-jsonl > "$O/bench_c3.json" 2> "$O/bench_c3.err"
echo "bench c3 $? $(python scripts/roofline_line.py "$O/bench_c3.json" 2>&1 | tail -1)" >> "$O/status"
cat "$O/status"
