#!/bin/bash
# One gpurun call: parity tests, smoke, a bench line, the ncu launch list of
# the same bench command and one `ncu --set full` capture of the top kernel.
#   gpurun --timeout 2400 -- bash scripts/gpu_check.sh [kernel-regex] [tag]
# Everything lands in gpurun_out/<tag>/.
set -u
K=${1:-k_downsweep}
TAG=${2:-run}
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$O/gpu.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest_gpu exit $?" >> "$O/status.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1
echo "smoke exit $?" >> "$O/status.txt"
timeout 900 python bench.py --steps 10 --warmup 3 > "$O/bench.json" 2> "$O/bench.err"
echo "bench exit $?" >> "$O/status.txt"
BC="python bench.py --steps 2 --warmup 3 --no-cpu"
timeout 600 $BC > "$O/plain.log" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$O/launches.csv" $BC > "$O/ncu_launches.log" 2>&1
echo "ncu launches exit $?" >> "$O/status.txt"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 2 -c 3 \
    -o "$O/prof" $BC > "$O/ncu_full.log" 2>&1
echo "ncu full exit $?" >> "$O/status.txt"
cat "$O/status.txt"
