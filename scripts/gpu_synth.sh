#!/bin/bash
set -u
O=gpurun_out/${1:-synth}
mkdir -p "$O"
timeout 600 python -m pytest tests/test_gpu_synth.py -x -q > "$O/pytest_synth.log" 2>&1
echo "pytest synth $?" >> "$O/status"
timeout 900 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest gpu $?" >> "$O/status"
cat "$O/status"
