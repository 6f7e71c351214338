#!/bin/bash
# ncu launch list of the default bench command + one `ncu --set full`
# capture of a kernel (after the plain command exits 0).
#   gpurun -- bash scripts/ncu_head.sh <kernel-regex> <tag>
K=${1:-k_scatter}; O=gpurun_out/${2:-ncu}; mkdir -p $O
BC="python bench.py --steps 2 --warmup 3 --no-cpu"
timeout 600 $BC > "$O/plain.log" 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file "$O/launches.csv" $BC > "$O/ncu_launches.log" 2>&1
echo "ncu launches exit $?" >> "$O/status.txt"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 2 -c 3 \
    -o "$O/prof" $BC > "$O/ncu_full.log" 2>&1
echo "ncu full exit $?" >> "$O/status.txt"
