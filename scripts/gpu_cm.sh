#!/bin/bash
# k_chunkmax block size A/B on the C2 store + the launch list after the
# fetch / pack changes.
set -u
O=gpurun_out/${1:-cm}
mkdir -p "$O"
for T in 512 256 128; do
  CSG_CM_THREADS=$T TAG=cm$T timeout 300 python scripts/kbench.py > "$O/kbench_cm$T.txt" 2>&1
  echo "cm $T $? $(grep k_chunkmax $O/kbench_cm$T.txt)" >> "$O/status"
done
BC="python bench.py --steps 2 --warmup 3 --no-cpu --no-jsonl"
timeout 600 $BC > "$O/plain.log" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$O/launches.csv" $BC > "$O/ncu_launches.log" 2>&1
echo "ncu launches $?" >> "$O/status"
cat "$O/status"
