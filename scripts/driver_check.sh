#!/bin/bash
# What the round-end driver runs on one GPU: the GPU suite, smoke, the
# default bench line and the reference arm.
set -u
O=gpurun_out/${1:-driver}
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$O/gpu.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest_gpu $?" >> "$O/status"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1
echo "smoke $?" >> "$O/status"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > "$O/bench.json" 2> "$O/bench.err"
echo "bench $? $(python scripts/roofline_line.py "$O/bench.json" 2>&1 | tail -1)" >> "$O/status"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > "$O/bench_ref.json" 2> "$O/bench_ref.err"
echo "bench ref $? $(head -c 300 $O/bench_ref.json)" >> "$O/status"
cat "$O/status"
