#!/bin/bash
# A/B of index-build variants on one GPU: parity of the TMA-tensor scatter
# (CSG_SCATTER_CFG=3) and bench lines per variant.
#   gpurun --timeout 1800 -- bash scripts/ab_index.sh <tag>
set -u
O=gpurun_out/${1:-ab}
mkdir -p "$O"
CSG_SCATTER_CFG=3 timeout 600 python -m pytest tests/test_gpu_index.py tests/test_gpu_catalog.py -x -q > "$O/pytest_cfg3.log" 2>&1
echo "pytest cfg3 $?" >> "$O/status"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > "$O/bench_base.json" 2> "$O/bench_base.err"
echo "bench base $?" >> "$O/status"
CSG_SCATTER_CFG=3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > "$O/bench_cfg3.json" 2> "$O/bench_cfg3.err"
echo "bench cfg3 $?" >> "$O/status"
CSG_CM_THREADS=512 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > "$O/bench_cm512.json" 2> "$O/bench_cm512.err"
echo "bench cm512 $?" >> "$O/status"
if grep -q "bench cfg3 0" "$O/status"; then
  CSG_SCATTER_CFG=3 timeout 600 ncu --set full --clock-control none --import-source on \
      -k "regex:k_scatter" -s 2 -c 2 -o "$O/prof_cfg3" \
      python bench.py --steps 2 --warmup 3 --no-cpu > "$O/ncu.log" 2>&1
  echo "ncu $?" >> "$O/status"
fi
cat "$O/status"
