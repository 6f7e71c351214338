#!/bin/bash
# C3 bench under each path knob (default, then one slow path at a time).
#   gpurun --timeout 1800 -- bash scripts/bisect_c3.sh <tag>
set -u
O=gpurun_out/${1:-bis}
mkdir -p "$O"
timeout 600 python -m pytest tests/test_gpu_selfev.py -x -q > "$O/pytest.log" 2>&1
echo "pytest $?" >> "$O/status"
for K in NONE CSG_SF_SLOW CSG_SL_SERIAL CSG_ITER_PER_TRIP CSG_FLOW_SCAN; do
  env $( [ $K != NONE ] && echo "$K=1" ) CSG_DEBUG_RETRY=1 timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-jsonl > "$O/c3_$K.json" 2> "$O/c3_$K.err"
  echo "c3 $K $? $(python scripts/roofline_line.py "$O/c3_$K.json" 2>&1 | tail -1)" >> "$O/status"
done
cat "$O/status"
