#!/bin/bash
O=gpurun_out/${1:-early}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/status
for v in 0 1; do
  if [ $v = 1 ]; then export CSG_STATS_FETCH=1; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-jsonl > $O/bench_statsfetch$v.json 2> $O/bench_statsfetch$v.err
  echo "bench statsfetch=$v $? $(python scripts/roofline_line.py $O/bench_statsfetch$v.json 2>&1 | tail -1)" >> $O/status
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-jsonl > $O/bench2_statsfetch$v.json 2> $O/bench2_statsfetch$v.err
  echo "bench statsfetch=$v $? $(python scripts/roofline_line.py $O/bench2_statsfetch$v.json 2>&1 | tail -1)" >> $O/status
done
unset CSG_STATS_FETCH
timeout 600 python scripts/timeline.py > $O/tl.out 2> $O/tl.err
