#!/bin/bash
# A/B of index-build variants on one GPU: parity of a CSG_SCATTER_CFG variant
# and bench lines for the default and the variant, then an ncu capture of
# the variant's k_scatter.
#   gpurun --timeout 1800 -- bash scripts/ab_index.sh <tag> <cfg>
set -u
O=gpurun_out/${1:-ab}
V=${2:-4}
mkdir -p "$O"
CSG_SCATTER_CFG=$V timeout 600 python -m pytest tests/test_gpu_index.py tests/test_gpu_catalog.py -x -q > "$O/pytest_cfg$V.log" 2>&1
echo "pytest cfg$V $?" >> "$O/status"
for i in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > "$O/bench_base$i.json" 2> "$O/bench_base$i.err"
echo "bench base $?" >> "$O/status"
CSG_SCATTER_CFG=$V timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > "$O/bench_cfg$V.$i.json" 2> "$O/bench_cfg$V.$i.err"
echo "bench cfg$V $?" >> "$O/status"
done
if grep -q "bench cfg$V 0" "$O/status"; then
  CSG_SCATTER_CFG=$V timeout 600 ncu --set full --clock-control none --import-source on \
      -k "regex:k_scatter" -s 2 -c 2 -o "$O/prof_cfg$V" \
      python bench.py --steps 2 --warmup 3 --no-cpu > "$O/ncu.log" 2>&1
  echo "ncu $?" >> "$O/status"
fi
cat "$O/status"
