#!/bin/bash
# Round check on one GPU: full GPU suite, smoke, C2 bench (default line),
# C3 and C4 bench lines.
#   gpurun --timeout 3000 -- bash scripts/gpu_full.sh <tag>
set -u
O=gpurun_out/${1:-full}
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$O/gpu.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest_gpu $?" >> "$O/status"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1
echo "smoke $?" >> "$O/status"
timeout 900 python bench.py --steps 20 --warmup 5 > "$O/bench.json" 2> "$O/bench.err"
echo "bench c2 $? $(python scripts/roofline_line.py "$O/bench.json" 2>&1 | tail -1)" >> "$O/status"
timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu --no-jsonl > "$O/bench_c3.json" 2> "$O/bench_c3.err"
echo "bench c3 $? $(python scripts/roofline_line.py "$O/bench_c3.json" 2>&1 | tail -1)" >> "$O/status"
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu > "$O/bench_c4.json" 2> "$O/bench_c4.err"
echo "bench c4 $? $(python scripts/roofline_line.py "$O/bench_c4.json" 2>&1 | tail -1)" >> "$O/status"
cat "$O/status"
