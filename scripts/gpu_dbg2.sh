#!/bin/bash
# k_exonerate phase breakdown on C2, then the ncu launch list + one full
# capture of k_scatter for profiles/.
set -u
O=gpurun_out/${1:-dbg2}
mkdir -p "$O"
CSG_DEBUG_EXO=1 timeout 300 python scripts/kbench.py > "$O/exo_debug_c2.txt" 2>&1
echo "exo debug c2 $?" >> "$O/status"
BC="python bench.py --steps 2 --warmup 3 --no-cpu --no-jsonl"
timeout 600 $BC > "$O/plain.log" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$O/launches.csv" $BC > "$O/ncu_launches.log" 2>&1
echo "ncu launches $?" >> "$O/status"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_scatter" -s 2 -c 2 \
    -o "$O/prof" $BC > "$O/ncu_full.log" 2>&1
echo "ncu full $?" >> "$O/status"
cat "$O/status"
