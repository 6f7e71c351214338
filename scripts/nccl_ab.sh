#!/bin/bash
# NCCL protocol A/B for the sharded C2 replay at N = <gpus>.
set -u
O=gpurun_out/${1:-nccl}
mkdir -p "$O"
G=$(nvidia-smi -L | wc -l)
run() {
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
      --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $G --steps 20 \
      --warmup 5 --no-jsonl > "$O/bench_$1.json" 2> "$O/bench_$1.err"
  echo "$1 $? $(python scripts/roofline_line.py $O/bench_$1.json 2>&1 | tail -1)" >> "$O/status"
}
run default 29501
NCCL_PROTO=LL128 run ll128 29502
NCCL_PROTO=LL run ll 29503
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING run debug 29504
grep -i "nvls\|algo\|proto" "$O/bench_debug.err" | head -40 > "$O/nccl_info.txt"
cat "$O/status"
