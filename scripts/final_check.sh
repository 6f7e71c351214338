#!/bin/bash
# Round-end check on HEAD (4 GPUs): the driver's one-GPU tiers, then the
# multi-GPU bench lines.   gpurun --gpus 4 -- bash scripts/final_check.sh <tag>
T=${1:-final}
bash scripts/driver_check.sh $T
O=gpurun_out/$T
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 10 \
      --warmup 3 > "$O/bench_n$N.json" 2> "$O/bench_n$N.err"
  echo "bench c2 n$N $? $(python scripts/roofline_line.py "$O/bench_n$N.json" 2>&1 | tail -1)" >> "$O/status"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 4 --workload c4 --steps 5 \
    --warmup 3 > "$O/bench_c4_n4.json" 2> "$O/bench_c4_n4.err"
echo "bench c4 n4 $? $(python scripts/roofline_line.py "$O/bench_c4_n4.json" 2>&1 | tail -1)" >> "$O/status"
