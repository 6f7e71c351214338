#!/bin/bash
# A/B of several CSG_SCATTER_CFG variants on one GPU: index + catalog parity
# per variant, then alternating bench lines (the roofline kernel's launch
# time), then one ncu --set full capture of k_place/k_scatter per variant.
#   gpurun --timeout 1800 -- bash scripts/ab_multi.sh <tag> <cfg> [<cfg> ...]
set -u
O=gpurun_out/${1:-ab}
shift
mkdir -p "$O"
for V in 0 "$@"; do
  CSG_SCATTER_CFG=$V timeout 600 python -m pytest tests/test_gpu_index.py tests/test_gpu_catalog.py -x -q > "$O/pytest_cfg$V.log" 2>&1
  echo "pytest cfg$V $?" >> "$O/status"
done
for i in 1 2; do
  for V in 0 "$@"; do
    CSG_SCATTER_CFG=$V timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > "$O/bench_cfg$V.$i.json" 2> "$O/bench_cfg$V.$i.err"
    echo "bench cfg$V $? $(python scripts/roofline_line.py "$O/bench_cfg$V.$i.json" 2>&1)" >> "$O/status"
  done
done
for V in 0 "$@"; do
  CSG_SCATTER_CFG=$V timeout 600 ncu --set full --clock-control none --import-source on \
      -k "regex:k_scatter|k_place" -s 1 -c 1 -o "$O/prof_cfg$V" \
      python bench.py --steps 2 --warmup 3 --no-cpu > "$O/ncu_cfg$V.log" 2>&1
  echo "ncu cfg$V $?" >> "$O/status"
done
cat "$O/status"
