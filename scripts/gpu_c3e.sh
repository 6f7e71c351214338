#!/bin/bash
set -u
O=gpurun_out/${1:-c3e}
mkdir -p "$O"
timeout 420 python -m pytest tests/test_gpu_selfev.py -x -q > "$O/pytest_selfev.log" 2>&1
echo "pytest selfev $?" >> "$O/status"
CSG_DEBUG_SF=1 timeout 500 python scripts/c3_paths.py > "$O/c3_paths.json" 2> "$O/c3_paths.err"
echo "c3_paths $? $(cat $O/c3_paths.json | tail -1)" >> "$O/status"
timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-jsonl > "$O/bench_c3.json" 2> "$O/bench_c3.err"
echo "bench c3 $? $(python scripts/roofline_line.py "$O/bench_c3.json" 2>&1 | tail -1)" >> "$O/status"
timeout 600 python -m pytest tests/test_gpu_catalog.py -x -q > "$O/pytest_catalog.log" 2>&1
echo "pytest catalog $?" >> "$O/status"
cat "$O/status"
