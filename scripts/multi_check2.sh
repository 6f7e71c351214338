#!/bin/bash
# Multi-GPU round check: sharded parity, C2 weak scaling at N = 2 and 4, the
# C4 job and the C3 shape (weak: DP x N) at N = 4.
#   gpurun --gpus 4 --timeout 3000 -- bash scripts/multi_check2.sh <tag>
set -u
O=gpurun_out/${1:-multi}
mkdir -p "$O"
G=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > "$O/pytest_multi.log" 2>&1
echo "pytest multi $?" >> "$O/status"
for N in 2 $G; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 10 \
      --warmup 3 > "$O/bench_n$N.json" 2> "$O/bench_n$N.err"
  echo "bench c2 n$N $? $(python scripts/roofline_line.py "$O/bench_n$N.json" 2>&1 | tail -1)" >> "$O/status"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
    --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus $G --workload c4 --steps 5 \
    --warmup 3 > "$O/bench_c4_n$G.json" 2> "$O/bench_c4_n$G.err"
echo "bench c4 n$G $? $(python scripts/roofline_line.py "$O/bench_c4_n$G.json" 2>&1 | tail -1)" >> "$O/status"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
    --master-addr 127.0.0.1 --master-port 29700 bench.py --gpus $G --workload c3 --steps 3 \
    --warmup 3 --no-jsonl > "$O/bench_c3_n$G.json" 2> "$O/bench_c3_n$G.err"
echo "bench c3 n$G $? $(python scripts/roofline_line.py "$O/bench_c3_n$G.json" 2>&1 | tail -1)" >> "$O/status"
cat "$O/status"
