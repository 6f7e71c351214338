#!/bin/bash
# Straggler-path check on one GPU: self-evidence + catalog parity, C3 default
# vs serial paths, C3 bench, the C5 slow-PCIe case with a timeline.
O=gpurun_out/${1:-coh}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_selfev.py tests/test_gpu_catalog.py -x -q > $O/pytest.log 2>&1; echo "pytest $?" >> $O/status
timeout 900 python scripts/c3_paths.py > $O/c3_paths.json 2> $O/c3_paths.err; echo "c3_paths $? $(tail -c 400 $O/c3_paths.json)" >> $O/status
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-jsonl > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 $? $(python scripts/roofline_line.py $O/bench_c3.json 2>&1 | tail -1)" >> $O/status
timeout 300 python scripts/sweep_c5.py --cases slow_pcie --timeline slow_pcie --cpu-replay "" --cpu-cap 1 > $O/c5_n1.json 2> $O/c5_n1.err; echo "c5 $?" >> $O/status
