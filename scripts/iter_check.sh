#!/bin/bash
set -u
O=gpurun_out/iter1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_selfev.py tests/test_gpu_catalog.py tests/test_gpu_multi.py -x -q > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status
timeout 300 python scripts/sweep_c5.py --cases slow_pcie,nic_flap --timeline slow_pcie --cpu-replay "" --cpu-cap 1 > $O/c5_n1.json 2> $O/c5_n1.err; echo "n1 $?" >> $O/status
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 scripts/sweep_c5.py --timeline slow_pcie > $O/c5_n4.json 2> $O/c5_n4.err; echo "n4 $?" >> $O/status
