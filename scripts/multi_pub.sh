#!/bin/bash
# Sharded trip publish: multi-GPU parity + C2 N=2/4 with and without it.
O=gpurun_out/${1:-mpub}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $O/pytest_multi.log 2>&1; echo "pytest multi $?" >> $O/status
for v in 0 1; do
  if [ $v = 1 ]; then export CSG_TRIG_FETCH=1; fi
  for N in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29500 + N + 10 * v)) bench.py --gpus $N --steps 10 --warmup 3 --no-jsonl \
        > $O/bench_n${N}_f$v.json 2> $O/bench_n${N}_f$v.err
    echo "fetch=$v n$N $? $(python scripts/roofline_line.py $O/bench_n${N}_f$v.json 2>&1 | tail -1)" >> $O/status
  done
done
