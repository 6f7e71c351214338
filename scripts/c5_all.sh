#!/bin/bash
# C5 fault sweep at N = 1 (with the reference analyzer's windows and whole
# replays), 2 and 4 GPUs:  gpurun --gpus 4 -- bash scripts/c5_all.sh <tag>
O=gpurun_out/${1:-c5}; mkdir -p $O
timeout 1300 python scripts/sweep_c5.py > $O/c5_n1.json 2> $O/c5_n1.err; echo "n1 $?" >> $O/status
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2961$n scripts/sweep_c5.py > $O/c5_n$n.json 2> $O/c5_n$n.err; echo "n$n $?" >> $O/status
done
