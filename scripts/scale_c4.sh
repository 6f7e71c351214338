#!/bin/bash
# C4 (fixed 65,536-rank job) at N = 4, 2, 1 and the C2 weak-scaling lines at
# N = 2, 4 on one 4-GPU box:  gpurun --gpus 4 -- bash scripts/scale_c4.sh <tag>
set -u
O=gpurun_out/${1:-scale}
mkdir -p "$O"
run() {  # run <n> <workload> <name>
  if [ "$1" = 1 ]; then
    timeout 1500 python bench.py --steps 5 --warmup 3 --workload "$2" --no-cpu \
      > "$O/$3.json" 2> "$O/$3.err"
  else
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" \
      --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus "$1" --steps 5 \
      --warmup 3 --workload "$2" > "$O/$3.json" 2> "$O/$3.err"
  fi
  echo "$3 exit $?" >> "$O/status.txt"
}
run 4 c4 c4_n4
run 2 c4 c4_n2
run 1 c4 c4_n1
run 2 c2 c2_n2
run 4 c2 c2_n4
cat "$O/status.txt"
