#!/bin/bash
# Side-stream successor all-reduce: sharded parity + C2 at N=<gpus> with and
# without the overlap (CSG_NO_COMM_OVERLAP=1).
set -u
O=gpurun_out/${1:-ovl}
mkdir -p "$O"
G=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > "$O/pytest_multi.log" 2>&1
echo "pytest multi $?" >> "$O/status"
for i in 1 2; do
  for V in 0 1; do
    if [ $V = 1 ]; then export CSG_NO_COMM_OVERLAP=1; else unset CSG_NO_COMM_OVERLAP; fi
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29600 + V + 2 * i)) bench.py --gpus $G --steps 20 \
        --warmup 5 --no-jsonl > "$O/bench_ovl$V.$i.json" 2> "$O/bench_ovl$V.$i.err"
    echo "no_overlap=$V $? $(python scripts/roofline_line.py $O/bench_ovl$V.$i.json 2>&1 | tail -1)" >> "$O/status"
  done
done
unset CSG_NO_COMM_OVERLAP
cat "$O/status"
